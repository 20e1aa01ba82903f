#!/bin/bash
# Bench lines for every BASELINE config on one B200 (run through gpurun), plus the GPU
# test suite: gpurun_out/${PROF_OUT}/bench_cN.log (JSON line) and gputest.log.
set -u
out=gpurun_out/${PROF_OUT:-all_r02}
mkdir -p $out
if [ "${SKIP_TESTS:-0}" = 0 ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > $out/gputest.log 2>&1
  echo "gpu tests rc=$?" >> $out/status.txt
fi
for c in ${CONFIGS:-c4 c2 c1 c5 c3}; do
  timeout 1500 python bench.py --config $c > $out/bench_$c.log 2> $out/bench_$c.err
  echo "bench $c rc=$?" >> $out/status.txt
done
