LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/keep.so
for v in ${1//,/ }; do cp tools/variants/$v.so $LIB; echo "== $v $(bash tools/bracket_time.sh | head -1 | awk -F, '{print $NF}')"; done
cp /tmp/keep.so $LIB
bash tools/variant_bench.sh ${1} --steps 10 --warmup 3
