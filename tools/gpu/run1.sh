# GPU session script: tests, smoke, C2 bench, one traced C2 batch, DADD latency probe
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -O3 -o /tmp/dadd_lat tools/probe/dadd_lat.cu && /tmp/dadd_lat > gpurun_out/dadd_lat.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; tail -5 gpurun_out/bench_c2.log; cat gpurun_out/bench_c2.json
DLP_LP_TRACE=gpurun_out/trace_c2.txt timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/bench_trace.json 2>gpurun_out/bench_trace.log
python tools/lp_trace.py gpurun_out/trace_c2.txt 1 > gpurun_out/trace_c2_summary.txt 2>&1; cat gpurun_out/trace_c2_summary.txt
