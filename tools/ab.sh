#!/bin/bash
# A/B of the C1 step time: build/libdelta_old.so vs the in-tree library, alternating runs
for i in 1 2 3; do
  echo "old: $(DELTA_LIB_PATH=$PWD/build/libdelta_old.so python tools/step_time.py "$@" 2>&1 | tail -1)"
  echo "new: $(python tools/step_time.py "$@" 2>&1 | tail -1)"
done
