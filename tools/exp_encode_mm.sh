#!/bin/bash
# like exp_encode.sh, but runs tools/diag_encode_mismatch.py (parity on the mixed 2-pass / 3-pass data)
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
  (cd .. && timeout 300 python tools/diag_encode_mismatch.py 2>&1 | head -4 >> $out/results.txt)
done
cat ../$out/results.txt
