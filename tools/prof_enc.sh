#!/bin/bash
# Encoder profiling on one B200 (run through gpurun): timing runs first, then the ncu
# launch list and one --set full capture per tensor-core encoder kernel.
set -u
out=gpurun_out/${1:-prof_enc}
mkdir -p $out
timeout 600 python tools/diag_encode_gpu.py > $out/enc_c4.log 2>&1
echo "enc c4 rc=$?" >> $out/status.txt
timeout 600 python tools/diag_encode_c3b.py > $out/enc_c3.log 2>&1
echo "enc c3 rc=$?" >> $out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $out/launches_c3.csv \
  python tools/diag_encode_c3b.py > $out/ncu_launch_c3.log 2>&1
echo "launch list c3 rc=$?" >> $out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tck_kernel -s 1 -c 1 \
  -o $out/ncu_tck_c3 python tools/diag_encode_c3b.py > $out/ncu_tck.log 2>&1
echo "ncu tck rc=$?" >> $out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tc_kernel -s 1 -c 1 \
  -o $out/ncu_tc_c4 python tools/diag_encode_gpu.py 2000000 > $out/ncu_tc.log 2>&1
echo "ncu tc rc=$?" >> $out/status.txt
