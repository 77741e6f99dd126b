LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/keep.so
for v in ${1//,/ }; do cp tools/variants/$v.so $LIB; echo "== $v $(python tools/parareal_time2d.py 4 2>&1 | grep -E 'time-to-tol' | cut -c1-60) $(python tools/parareal_time2d.py 4 2>&1 | grep stats | grep -o "'pcg_iterations': [0-9]*")"; done
cp /tmp/keep.so $LIB
