#!/bin/bash
# tests + bench + latency trace.  Usage: gpurun -- bash tools/gpu_trace.sh TAG [tests|notests]
set -u
TAG=${1:-t}; TESTS=${2:-tests}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$TESTS" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -5 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -3 $OUT/bench.err
timeout 300 python tools/trace_probe.py > $OUT/trace.txt 2>&1; echo "trace exit $?" >> $OUT/trace.txt
cat $OUT/trace.txt
