set -x
mkdir -p gpurun_out
start=$(date +%s)
timeout 2400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
echo "reference arm wall $(( $(date +%s) - start )) s"
tail -5 gpurun_out/bench_ref.log; head -c 2500 gpurun_out/bench_ref.json
