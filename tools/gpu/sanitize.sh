set -x
mkdir -p gpurun_out
for cfg in "0 0" "8 24" "100000 100000"; do
  set -- $cfg
  DLP_LONG_ROW=$1 DLP_HUB_ROW=$2 timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python tests/_row_class_check.py 10 2>&1 | tail -3
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_reference_kats.py tests/test_harmonic.py -q -m gpu -p no:cacheprovider 2>&1 | tail -3
