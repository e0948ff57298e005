#!/bin/bash
# compute-sanitizer sweep (racecheck + memcheck) over representative GPU tests; one summary line
# per run -> gpurun_out/sanitizers.txt
out=gpurun_out/sanitizers.txt; mkdir -p gpurun_out; : > $out
run() {  # tool, test spec
  local log=gpurun_out/san_$1_$(echo "$2" | tr -c 'a-zA-Z0-9' '_').log
  timeout 900 compute-sanitizer --tool $1 python -m pytest $2 -x -q > $log 2>&1
  echo "$1 $2: $(grep -E 'SUMMARY' $log | tail -1) | pytest: $(grep -E 'passed|failed' $log | tail -1)" >> $out
}
for t in "tests/test_gpu_parity.py -k gs16" "tests/test_gpu_parity.py -k c0_page" "tests/test_gpu_raas.py -k 1" \
         "tests/test_gpu_quest.py -k d64" "tests/test_gpu_recall.py -k quest" "tests/test_gpu_prefill.py -k d64" \
         "tests/test_gpu_shard.py -k det_chunks_bitwise" "tests/test_gpu_parity.py -k heads_ragged" \
         "tests/test_gpu_parity.py -k ll_flags" "tests/test_gpu_parity.py -k ll_keys" "tests/test_gpu_prefill.py"; do
  run racecheck "$t"
done
for t in "tests/test_gpu_parity.py -k c0_page" "tests/test_gpu_shard.py -k det_chunks" "tests/test_gpu_raas.py -k 1" \
         "tests/test_gpu_prefill.py" "tests/test_gpu_quest.py -k d64" "tests/test_gpu_parity.py -k ll_flags" \
         "tests/test_gpu_parity.py -k ll_keys" "tests/test_gpu_parity.py -k heads_ragged"; do
  run memcheck "$t"
done
cat $out
