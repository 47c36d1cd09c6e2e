# A/B of LP kernel variants on C2 (short bench legs), then an ncu source profile of the current kernel
set -x
mkdir -p gpurun_out
for v in head new lrpt32; do
  DLP_LIB_PATH=variants/lib_$v.so timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.log
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', d['value'], d['e2e']['value'], d['step_wall_ms']['lp_kernel'])"
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/lp_new python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/ncu_new.log 2>&1
tail -3 gpurun_out/ncu_new.log
