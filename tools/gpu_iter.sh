#!/bin/bash
# Iteration loop on one box: GPU parity suite, bench, latency trace.
# Usage: gpurun -- bash tools/gpu_iter.sh TAG [tests|notests] [trace|notrace] [extra pytest -k expr]
set -u
TAG=${1:-i}; TESTS=${2:-tests}; TRACE=${3:-trace}; KEXPR=${4:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$TESTS" = tests ]; then
  if [ -n "$KEXPR" ]; then
    timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  else
    timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  fi
  tail -15 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -3 $OUT/bench.err
if [ "$TRACE" = trace ]; then
  timeout 300 python tools/trace_probe.py > $OUT/trace.txt 2>&1; echo "trace exit $?" >> $OUT/trace.txt
  grep -E "select L|span|L 0:|L 3:|L 5:|L31:|exit" $OUT/trace.txt
fi
