# final round-end style session: tests, smoke, the driver's two arms, default bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
bash tools/gpu/driver_seq.sh
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; tail -1 gpurun_out/bench_c2.log; head -c 400 gpurun_out/bench_c2.json
