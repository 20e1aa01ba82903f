#!/bin/bash
# Encoder timing experiments on the GPU box: rebuilds pqk_encode_tc.o with -DENC_EXP=<mask>
# (and any extra -D flags given after the mask, comma separated), relinks the library and
# times config-4 encoding.  usage: bash tools/exp_encode.sh out_dir "0" "1" "2" "4,-DENC_XST=5" ...
set -u
out=gpurun_out/$1; shift
mkdir -p $out
cd paper_1709_03708_b200
for spec in "$@"; do
  mask=${spec%%,*}; extra=""
  if [[ "$spec" == *,* ]]; then extra=$(echo "${spec#*,}" | tr ',' ' '); fi
  nvcc -c csrc/pqk_encode_tc.cu -o _obj/pqk_encode_tc.o -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I ../include -I csrc \
    -gencode arch=compute_100a,code=sm_100a -DENC_EXP=$mask $extra || { echo "build failed $spec" >> ../$out/results.txt; continue; }
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o libpqk_b200.so _obj/*.o -cudart static
  echo "== ENC_EXP=$mask $extra" >> ../$out/results.txt
  (cd .. && timeout 300 python tools/diag_encode_gpu.py 2>&1 | grep -E "encode|flagged|mismatch" >> $out/results.txt)
done
cat ../$out/results.txt
