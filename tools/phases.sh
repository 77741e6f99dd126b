# build a -DPF_PHASE_TIMING variant of the library in a scratch copy and print the phase breakdown
set -e
mkdir -p /tmp/ptime && cp -r paper_2510_11023_b200 include /tmp/ptime/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPF_PHASE_TIMING -Xcompiler -fPIC -shared \
  -o /tmp/ptime/paper_2510_11023_b200/libparafrac_b200.so /tmp/ptime/paper_2510_11023_b200/csrc/pf_api.cu
sed 's#/root/repo#/tmp/ptime#' tools/phases.py > /tmp/ptime/phases.py
python /tmp/ptime/phases.py ${1:-3}
