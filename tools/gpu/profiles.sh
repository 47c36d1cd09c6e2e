# profiles of the current kernels: LP (C2, C4), kNN screen, launch list; C3 and C4 bench lines
set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-knn --no-itlp --no-readback"
timeout 1200 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/r02_lp_c2 $B --steps 1 --warmup 3 > gpurun_out/ncu_lp_c2.log 2>&1; tail -1 gpurun_out/ncu_lp_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv $B --steps 2 --warmup 3 > gpurun_out/launch_c2.log 2>&1; tail -1 gpurun_out/launch_c2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_knn_screen -s 2 -c 1 -o gpurun_out/r02_knn python bench.py --no-cpu-baseline --no-itlp --no-readback --steps 1 --warmup 3 > gpurun_out/ncu_knn.log 2>&1; tail -1 gpurun_out/ncu_knn.log
timeout 1800 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; tail -2 gpurun_out/bench_c3.log; head -c 600 gpurun_out/bench_c3.json; echo
timeout 2400 python bench.py --config c4 --no-knn --no-itlp --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; tail -2 gpurun_out/bench_c4.log; head -c 600 gpurun_out/bench_c4.json; echo
timeout 1800 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/r02_lp_c4 python bench.py --config c4 --no-cpu-baseline --no-knn --no-itlp --no-readback --steps 1 --warmup 3 > gpurun_out/ncu_lp_c4.log 2>&1; tail -1 gpurun_out/ncu_lp_c4.log
