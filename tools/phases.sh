# per-phase cycle breakdown of slice 0 (a -DPF_PHASE_TIMING library in a scratch copy):
#   tools/phases.sh build      (here: nvcc into tools/variants/phase.so, travels with gpurun)
#   tools/phases.sh [config]   (on the GPU box)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = "build" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPF_PHASE_TIMING -Xcompiler -fPIC -shared \
    -o "$ROOT/tools/variants/phase.so" "$ROOT/paper_2510_11023_b200/csrc/pf_api.cu"
  exit 0
fi
rm -rf /tmp/ptime && mkdir -p /tmp/ptime && cp -r "$ROOT/paper_2510_11023_b200" "$ROOT/include" /tmp/ptime/
cp "$ROOT/tools/variants/${PHASE_SO:-phase}.so" /tmp/ptime/paper_2510_11023_b200/libparafrac_b200.so
SCRIPT=${PHASE_SCRIPT:-tools/phases.py}
sed "s#/root/repo#/tmp/ptime#" "$ROOT/$SCRIPT" > /tmp/ptime/phases.py
# one launch (no head start): slice 0 is block 0 of the sweep, the only CTA the timers follow
PF_NO_HEADSTART=1 python /tmp/ptime/phases.py ${1:-3}
