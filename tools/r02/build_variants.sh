#!/bin/bash
# build A/B variants in parallel: tools/r02/build_variants.sh "name1:-DX=1 -DY=2" "name2:-DZ=1" ...
cd "$(dirname "$0")/../.."
mkdir -p tools/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $flags \
      -o tools/variants/$name.so paper_2510_11023_b200/csrc/pf_api.cu 2>&1 | grep -E " error" ; echo "built $name" ) &
done
wait
