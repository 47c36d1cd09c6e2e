# usage: bash tools/gpu/ab.sh "spec ..." [tests] [config]
#   spec = <lib>[:VAR=val[,VAR=val]]  (lib: main = in-tree library, else variants/lib_<lib>.so)
set -x
mkdir -p gpurun_out
CFG=${3:-c2}
if [ "$2" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -5 gpurun_out/pytest_gpu.txt
fi
for spec in $1; do
  v=${spec%%:*}; envs=""; [ "$v" != "$spec" ] && envs=${spec#*:}
  if [ "$v" = "main" ]; then L=paper_2604_06596_b200/libdynlp_b200.so; else L=variants/lib_$v.so; fi
  tag=$(echo "$spec" | tr ':=,' '___')
  env DLP_LIB_PATH=$L $(echo $envs | tr ',' ' ') timeout 900 python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.log
  python -c "import json; d=json.load(open('gpurun_out/ab_$tag.json')); print('AB $CFG $spec', round(d['value'],2), round(d['e2e']['value'],2), d['step_wall_ms']['lp_kernel'])" || tail -5 gpurun_out/ab_$tag.log
done
