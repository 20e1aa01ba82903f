#!/bin/bash
# K-streamed encoder on one B200 (run through gpurun): quick parity check, parity tests,
# timing, launch list, then (arg 2 = full) one ncu --set full capture of encode_tck_kernel
# at config 3's chunk shape.
set -u
out=gpurun_out/${1:-prof_tck}
mkdir -p $out
timeout 180 python tools/diag_encode_c3.py 20000 > $out/quick.log 2>&1
echo "quick rc=$?" >> $out/status.txt
tail -2 $out/quick.log
if ! grep -q "mismatch vs oracle on first 2000 : 0" $out/quick.log; then cat $out/status.txt; exit 1; fi
timeout 400 python -m pytest tests/test_gpu_encode_tc.py tests/test_gpu_kernels.py -m gpu -x -q > $out/tests.log 2>&1
echo "tests rc=$?" >> $out/status.txt
tail -3 $out/tests.log
timeout 600 python tools/diag_encode_c3b.py > $out/enc_c3.log 2>&1
PQK_ENCODE_TCK_PAIR=0 timeout 600 python tools/diag_encode_c3b.py > $out/enc_c3_nopair.log 2>&1; echo nopair; tail -2 $out/enc_c3_nopair.log
echo "enc c3 rc=$?" >> $out/status.txt
cat $out/enc_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $out/launches_c3.csv \
  python tools/diag_encode_c3b.py > $out/ncu_launch_c3.log 2>&1
echo "launch list c3 rc=$?" >> $out/status.txt
grep -E "encode_tck" $out/launches_c3.csv | awk -F'","' '{print $5, $NF}' | tail -3
if [ "${2:-full}" = "full" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tck_kernel -s 1 -c 1 \
  -o $out/ncu_tck_c3 python tools/diag_encode_c3b.py > $out/ncu_tck.log 2>&1
echo "ncu tck rc=$?" >> $out/status.txt
fi
cat $out/status.txt
