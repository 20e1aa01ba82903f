#!/bin/bash
# One ncu --set full capture (with SASS source counters) of encode_tc_kernel on config-4
# vectors; the raw and source pages are exported to CSV on the box (the .ncu-rep stays there).
set -u
out=gpurun_out/${1:-prof_enc_src}
mkdir -p $out
timeout 600 python tools/diag_encode_gpu.py > $out/enc_c4.log 2>&1
echo "enc c4 rc=$?" >> $out/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tc_kernel -s 1 -c 1 \
  -o $out/ncu_tc_c4 python tools/diag_encode_gpu.py 2000000 > $out/ncu_tc.log 2>&1
echo "ncu tc rc=$?" >> $out/status.txt
ncu -i $out/ncu_tc_c4.ncu-rep --page raw --csv > $out/ncu_tc_raw.csv 2>/dev/null
ncu -i $out/ncu_tc_c4.ncu-rep --page source --csv --print-source sass > $out/ncu_tc_sass.csv 2>/dev/null
echo "export rc=$?" >> $out/status.txt
