set -x
mkdir -p gpurun_out
free -g
timeout 1500 python -X faulthandler bench.py --config c4 --no-knn --no-itlp --no-readback --steps 2 --warmup 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "rc=$?"
free -g; dmesg 2>/dev/null | tail -5
grep -v "^\s*$" gpurun_out/bench_c4.log | tail -8; head -c 1200 gpurun_out/bench_c4.json; echo
