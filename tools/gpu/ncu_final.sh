set -x
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-knn --no-itlp --no-readback"
timeout 1200 ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_lp_fused -s 99 -c 1 -o gpurun_out/r02_lp_c2_final $B --steps 1 --warmup 3 > gpurun_out/ncu_lp_c2f.log 2>&1; tail -1 gpurun_out/ncu_lp_c2f.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2_final.csv $B --steps 2 --warmup 3 > gpurun_out/launch_c2f.log 2>&1; tail -1 gpurun_out/launch_c2f.log
