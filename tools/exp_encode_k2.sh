#!/bin/bash
# like exp_encode_k.sh, reporting the per-kernel times of the last config-3 chunk (ncu launch list)
set -u
out=gpurun_out/$1; shift
mkdir -p $out
cd paper_1709_03708_b200
for spec in "$@"; do
  extra=$(echo "$spec" | tr ',' ' ')
  nvcc -c csrc/pqk_encode_tc.cu -o _obj/pqk_encode_tc.o -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I ../include -I csrc \
    -gencode arch=compute_100a,code=sm_100a $extra || { echo "build failed $spec" >> ../$out/results.txt; continue; }
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o libpqk_b200.so _obj/*.o -cudart static
  echo "== $extra" >> ../$out/results.txt
  (cd .. && timeout 300 python tools/diag_encode_c3b.py 2>&1 | grep -E "^encode" | tail -1 >> $out/results.txt
   timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $out/l.csv python tools/diag_encode_c3b.py > /dev/null 2>&1
   grep -E "encode_tck|filter32_cand|exact_cand" $out/l.csv | tail -3 | awk -F'","' '{print substr($5,1,40), $NF}' >> $out/results.txt)
done
cat ../$out/results.txt
