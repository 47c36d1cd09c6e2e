set -x
bash tools/gpu/ab.sh "main long64 long160 scan16 scan256" notests c2
start=$(date +%s)
timeout 1500 python bench.py --config c4 --no-knn --no-itlp --no-readback --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
echo "c4 bench wall $(( $(date +%s) - start )) s"; grep -v "^\s*$" gpurun_out/bench_c4.log | tail -3; head -c 1500 gpurun_out/bench_c4.json; echo
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lp_fused -s 98 -c 1 -o gpurun_out/r02_lp_c4 python bench.py --config c4 --no-cpu-baseline --no-knn --no-itlp --no-readback --steps 1 --warmup 2 > gpurun_out/ncu_lp_c4.log 2>&1; grep -v "^\s*$" gpurun_out/ncu_lp_c4.log | tail -2
