set -x
timeout 600 python -m pytest tests/test_sharded.py -x -q -k nccl -p no:cacheprovider 2>&1 | grep -E "Error|passed|failed" | head -5
bash tools/gpu/ab.sh "main w64" notests c2
bash tools/gpu/ab.sh "main flat" notests c2b
