# build a macro variant of the library: tools/build_variant.sh NAME "-DFOO=1 ..."
NAME=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared $* \
  -o tools/variants/$NAME.so paper_2510_11023_b200/csrc/pf_api.cu 2>&1 | grep -E "error" 
