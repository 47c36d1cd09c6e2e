set -x
mkdir -p gpurun_out
cat /sys/fs/cgroup/memory.max /sys/fs/cgroup/memory/memory.limit_in_bytes 2>&1 | head -3
timeout 900 python tools/c4_stream_mem.py > gpurun_out/c4mem.txt 2>&1; echo "rc=$?"; tail -25 gpurun_out/c4mem.txt
