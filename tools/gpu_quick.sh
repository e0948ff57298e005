#!/bin/bash
# Quick GPU check: parity tests (optional), bench, per-role ncu capture.
# Usage: gpurun -- bash tools/gpu_quick.sh TAG [tests|notests] [ncu|noncu]
set -u
TAG=${1:-q}; TESTS=${2:-tests}; NCU=${3:-ncu}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ "$TESTS" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
cat $OUT/bench.json; tail -3 $OUT/bench.err
if [ "$NCU" = ncu ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'attn|select' --launch-skip 35 -c 12 \
      -o $OUT/probe python tools/kernel_probe.py > $OUT/ncu_probe.log 2>&1; echo "ncu exit $?" >> $OUT/ncu_probe.log
  tail -2 $OUT/ncu_probe.log
fi
