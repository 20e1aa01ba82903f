#!/bin/bash
# Round profile refresh on one B200 (run through gpurun): bench lines for every config,
# the config-2 launch list and one ncu --set full capture of the first-tier scan kernel.
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
out=gpurun_out/${PROF_OUT:-prof}
mkdir -p $out
for c in c2 c1 c5 c3 c4; do
  steps=5; [ $c = c4 ] && steps=2
  timeout 1500 python bench.py --config $c --steps $steps --warmup 3 > $out/bench_$c.log 2> $out/bench_$c.err
  echo "bench $c rc=$?" >> $out/status.txt
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $out/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
echo "launch list rc=$?" >> $out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hscan_kernel -s 2 -c 1 \
  -o $out/ncu_hscan_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $out/status.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vote_tc_kernel -s 2 -c 1 \
  -o $out/ncu_vote_tc_c2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_vote.log 2>&1
echo "ncu vote rc=$?" >> $out/status.txt
