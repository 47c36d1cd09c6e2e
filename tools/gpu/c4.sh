# C4 (10M x 64, k=16, binary): bench line and one ncu capture of k_lp_fused (working set >> L2)
set -x
mkdir -p gpurun_out
start=$(date +%s)
timeout 2000 python bench.py --config c4 --no-knn --no-itlp --no-readback --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
echo "c4 bench wall $(( $(date +%s) - start )) s"; tail -3 gpurun_out/bench_c4.log; head -c 1500 gpurun_out/bench_c4.json; echo
timeout 1200 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lp_fused -s 98 -c 1 -o gpurun_out/r02_lp_c4 python bench.py --config c4 --no-cpu-baseline --no-knn --no-itlp --no-readback --steps 1 --warmup 2 > gpurun_out/ncu_lp_c4.log 2>&1; tail -2 gpurun_out/ncu_lp_c4.log
