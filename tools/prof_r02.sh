#!/bin/bash
# Round-2 profile refresh on one B200 (run through gpurun): GPU tests, the default bench
# line (config-4 shard), its launch list and one ncu --set full capture of the first-tier
# scan kernel.  Each ncu command runs only after the same command exited 0 without ncu.
set -u
out=gpurun_out/${PROF_OUT:-prof_r02}
mkdir -p $out
if [ "${SKIP_TESTS:-0}" = 0 ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q > $out/gputest.log 2>&1
  echo "gpu tests rc=$?" >> $out/status.txt
fi
timeout 1200 python bench.py > $out/bench.log 2> $out/bench.err
echo "bench rc=$?" >> $out/status.txt
P="python bench.py --steps 1 --warmup 3 --no-extras --no-e2e --no-cpu-baseline --no-parity"
timeout 900 $P > $out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $out/launches_c4.csv \
  $P > $out/ncu_launch.log 2>&1
echo "launch list rc=$?" >> $out/status.txt
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-hscan8_kernel} -s 1 -c 1 \
  -o $out/ncu_scan_c4 $P > $out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $out/status.txt
