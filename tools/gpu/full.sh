# round-end style GPU session: tests, smoke, reference arm, bench, profiles
set -x
mkdir -p gpurun_out
{ nproc; free -g; } > gpurun_out/box.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
/usr/bin/time -v timeout 2400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; tail -3 gpurun_out/bench_ref.log; head -c 1500 gpurun_out/bench_ref.json
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; tail -3 gpurun_out/bench_c2.log; head -c 3000 gpurun_out/bench_c2.json
