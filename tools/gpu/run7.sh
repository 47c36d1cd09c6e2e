set -x
mkdir -p gpurun_out
for i in 1 2; do DLP_LONG_ROW=8 DLP_HUB_ROW=24 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -2; done
DLP_SM_MAX_NA=0 DLP_LONG_ROW=8 DLP_HUB_ROW=24 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -2
DLP_HUB_ROW=100000 DLP_LONG_ROW=8 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -2
DLP_HUB_ROW=24 DLP_LONG_ROW=100000 timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -2
timeout 300 python tests/_row_class_check.py 10 2>&1 | tail -2
DLP_LONG_ROW=8 DLP_HUB_ROW=24 timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tests/_row_class_check.py 10 > gpurun_out/racecheck.txt 2>&1; tail -30 gpurun_out/racecheck.txt
