set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; tail -1 gpurun_out/bench_c2.log; head -c 300 gpurun_out/bench_c2.json; echo
for m in 0 2; do DLP_L2_PERSIST=$m timeout 900 python bench.py --config c4 --no-knn --no-itlp --no-readback --steps 3 --warmup 3 > gpurun_out/c4_l2_$m.json 2> gpurun_out/c4_l2_$m.log; python -c "import json; d=json.load(open('gpurun_out/c4_l2_$m.json')); print('C4 L2 mode $m', d['value'], d['e2e']['value'])"; done
