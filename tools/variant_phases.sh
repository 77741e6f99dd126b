# phase breakdown (tools/phases.py) with each -DPF_PHASE_TIMING variant in $1
LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/lib_keep.so
for n in ${1//,/ }; do
  cp tools/variants/$n.so $LIB
  echo "== $n"; python tools/phases.py 3 2>&1 | tail -17
done
cp /tmp/lib_keep.so $LIB
