# per-warp timeline of a slice CTA (a -DPF_TRACE library in a scratch copy):
#   tools/r02/trace.sh build [extra nvcc flags]   (here: nvcc into tools/variants/trace.so)
#   tools/r02/trace.sh [config]                   (on the GPU box)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
if [ "$1" = "build" ]; then
  shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPF_TRACE -DPF_ONLY_S10 $* -Xcompiler -fPIC -shared \
    -o "$ROOT/tools/variants/${TRACE_SO:-trace}.so" "$ROOT/paper_2510_11023_b200/csrc/pf_api.cu"
  exit 0
fi
rm -rf /tmp/ptrace && mkdir -p /tmp/ptrace && cp -r "$ROOT/paper_2510_11023_b200" "$ROOT/include" /tmp/ptrace/
cp "$ROOT/tools/variants/${TRACE_SO:-trace}.so" /tmp/ptrace/paper_2510_11023_b200/libparafrac_b200.so
sed "s#/root/repo#/tmp/ptrace#" "$ROOT/tools/r02/trace.py" > /tmp/ptrace/trace.py
PF_NO_HEADSTART=1 python /tmp/ptrace/trace.py ${1:-3}
