LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/keep.so; cp tools/variants/ph0.so $LIB
python tools/phases.py 2 2>&1 | tail -16
python tools/phases.py 1 2>&1 | tail -16
cp /tmp/keep.so $LIB
