set -x
mkdir -p gpurun_out
for i in 1 2; do DLP_LONG_ROW=0 DLP_HUB_ROW=0 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -1; done
DLP_LONG_ROW=8 DLP_HUB_ROW=24 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/lp_view python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/ncu_view.log 2>&1
tail -2 gpurun_out/ncu_view.log
