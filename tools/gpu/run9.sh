set -x
mkdir -p gpurun_out
DLP_LONG_ROW=0 DLP_HUB_ROW=0 timeout 1200 compute-sanitizer --tool memcheck --print-limit 10 python tests/_row_class_check.py 10 > gpurun_out/sanitizer_rowclass00.txt 2>&1; grep -v "^=========     Host Frame" gpurun_out/sanitizer_rowclass00.txt | head -60
for i in 1 2 3; do DLP_LONG_ROW=0 DLP_HUB_ROW=0 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -1; done
