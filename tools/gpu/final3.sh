set -x
mkdir -p gpurun_out
bash tools/gpu/driver_seq.sh
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; tail -1 gpurun_out/bench_c2.log; head -c 300 gpurun_out/bench_c2.json
