# the driver's round-end sequence: reference arm, then the B200 arm, same window
set -x
mkdir -p gpurun_out
start=$(date +%s)
timeout 2400 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.log
echo "reference arm wall $(( $(date +%s) - start )) s"; tail -3 gpurun_out/drv_ref.log
start=$(date +%s)
timeout 2400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_b200.json 2> gpurun_out/drv_b200.log
echo "b200 arm wall $(( $(date +%s) - start )) s"; tail -2 gpurun_out/drv_b200.log
python -c "
import json; r=json.load(open('gpurun_out/drv_ref.json')); b=json.load(open('gpurun_out/drv_b200.json'))
print('ref', r['value'], r['cpu_baseline']['sample'][-80:])
print('b200', b['value'], b['e2e']['value'], b['roofline']['frac'], b.get('parity_with_reference_arm'), b['cpu_baseline']['parity_with_gpu'], b['cpu_baseline']['value'])
"
