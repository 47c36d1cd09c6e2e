# reference-arm hand-off labels for the driver's window (--steps 20 --warmup 5 -> t_h = 78)
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --make-handoff --steps 20 --warmup 5 2>&1 | tail -2
ls -la baseline/handoff/
cd baseline/handoff && for f in *.npz; do split -b 60m -d "$f" "../../gpurun_out/handoff_$f.part"; done; cd ../..
ls -la gpurun_out/
