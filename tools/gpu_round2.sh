#!/bin/bash
# Round evidence: parity suite, smoke, bench (with cpu baseline), ncu launch list of the bench,
# ncu --set full of the per-role kernels (tools/kernel_probe.py) and of the Quest kernels.
# Usage: gpurun --timeout 2400 -- bash tools/gpu_round2.sh TAG
set -u
TAG=${1:-r}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
tail -2 $OUT/bench.err
for c in c2 c3 c4; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 30 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "ncu list exit $?" >> $OUT/ncu_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'attn|select' --launch-skip 35 -c 12 \
    -o $OUT/probe python tools/kernel_probe.py > $OUT/ncu_probe.log 2>&1; echo "ncu probe exit $?" >> $OUT/ncu_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'quest|select' --launch-skip 60 -c 4 \
    -o $OUT/quest python tools/quest_probe.py > $OUT/ncu_quest.log 2>&1; echo "ncu quest exit $?" >> $OUT/ncu_quest.log
for f in ncu_bench ncu_probe ncu_quest; do tail -n 1 $OUT/$f.log; done
