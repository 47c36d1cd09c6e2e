set -x
mkdir -p gpurun_out
DLP_LONG_ROW=8 DLP_HUB_ROW=24 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tests/_row_class_check.py 10 > gpurun_out/sanitizer_rowclass.txt 2>&1; tail -40 gpurun_out/sanitizer_rowclass.txt
for v in main head; do
  if [ "$v" = "main" ]; then L=paper_2604_06596_b200/libdynlp_b200.so; else L=variants/lib_$v.so; fi
  DLP_LIB_PATH=$L DLP_LP_TRACE=gpurun_out/trace_$v.txt timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-knn --no-itlp --no-readback > /dev/null 2>&1
  python tools/lp_trace.py gpurun_out/trace_$v.txt 1 > gpurun_out/trace_${v}_summary.txt 2>&1; cat gpurun_out/trace_${v}_summary.txt
done
