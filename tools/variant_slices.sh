# per-slice PCG iterations / times (tools/slice_iters.py) for each tools/variants/<name>.so in $1
LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/lib_keep.so
for n in ${1//,/ }; do
  cp tools/variants/$n.so $LIB
  echo "== $n"; python tools/slice_iters.py 2>&1 | tail -4
done
cp /tmp/lib_keep.so $LIB
