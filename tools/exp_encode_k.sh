#!/bin/bash
# K-streamed encoder timing experiments on the GPU box: rebuilds pqk_encode_tc.o with
# -DENC_KEXP=<mask> (plus extra -D flags after the mask, comma separated), relinks the
# library and times config-3 encoding chunks (per-kernel times from an ncu launch list).
# usage: bash tools/exp_encode_k.sh out_dir "0" "1" "2" ...
set -u
out=gpurun_out/$1; shift
mkdir -p $out
cd paper_1709_03708_b200
for spec in "$@"; do
  mask=${spec%%,*}; extra=""
  if [[ "$spec" == *,* ]]; then extra=$(echo "${spec#*,}" | tr ',' ' '); fi
  nvcc -c csrc/pqk_encode_tc.cu -o _obj/pqk_encode_tc.o -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I ../include -I csrc \
    -gencode arch=compute_100a,code=sm_100a -DENC_KEXP=$mask $extra || { echo "build failed $spec" >> ../$out/results.txt; continue; }
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o libpqk_b200.so _obj/*.o -cudart static
  echo "== ENC_KEXP=$mask $extra" >> ../$out/results.txt
  (cd .. && timeout 300 python tools/diag_encode_c3b.py 2>&1 | grep -E "encode|tck" | tail -2 >> $out/results.txt)
done
cat ../$out/results.txt
