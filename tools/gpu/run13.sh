timeout 600 python -m pytest tests/test_sharded.py -x -q -k nccl -p no:cacheprovider 2>&1 | grep -E "InternalError|CudaError|passed|failed" | head -8
NCCL_DEBUG=WARN timeout 300 python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import test_sharded as t
t.test_nccl_in_handle_world1(0, 'blobs10', 'components')
print('ok')
" 2>&1 | tail -15
