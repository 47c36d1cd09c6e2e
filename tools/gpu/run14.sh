timeout 600 python -m pytest tests/test_sharded.py -x -q -k nccl -p no:cacheprovider 2>&1 | grep -E "InternalError|CudaError|passed|failed" | head -8
bash tools/gpu/ab.sh "main w64 hw256 hub256 hub1024" notests c2
