#!/bin/bash
# Runs the full-size C4 parity test with a host/device memory sampler beside it.
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests/test_baseline_parity.py -m gpu -q -k c4_first -s > gpurun_out/c4test.log 2>&1; echo "exit $?" >> gpurun_out/c4test.log ) &
job=$!
sleep 5
: > gpurun_out/c4mem.log
while kill -0 $job 2>/dev/null; do
  pid=$(pgrep -n -f "pytest tests/test_baseline_parity.py" || true)
  if [ -n "$pid" ]; then
    rss=$(grep -E "VmRSS|VmHWM" /proc/$pid/status 2>/dev/null | tr '\n' ' ')
    gpu=$(nvidia-smi --query-gpu=memory.used --format=csv,noheader 2>/dev/null)
    echo "$(date +%s) $rss gpu $gpu $(free -g | awk '/Mem/{print "hostfree " $4 " avail " $7}')" >> gpurun_out/c4mem.log
  fi
  sleep 3
done
wait $job
cat /sys/fs/cgroup/memory.max /sys/fs/cgroup/memory.peak 2>/dev/null >> gpurun_out/c4mem.log
tail -5 gpurun_out/c4mem.log
tail -15 gpurun_out/c4test.log
