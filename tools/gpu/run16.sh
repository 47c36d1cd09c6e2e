set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/lp_cur python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/ncu_cur.log 2>&1
tail -1 gpurun_out/ncu_cur.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 --csv --log-file gpurun_out/launches_cur.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/launch_cur.log 2>&1
DLP_LP_TRACE=gpurun_out/trace_cur.txt timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > /dev/null 2>&1
python tools/lp_trace.py gpurun_out/trace_cur.txt 1 > gpurun_out/trace_cur_summary.txt 2>&1; cat gpurun_out/trace_cur_summary.txt
