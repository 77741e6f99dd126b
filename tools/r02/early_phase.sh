set -e
ROOT=/root/repo
rm -rf /tmp/ptrace && mkdir -p /tmp/ptrace && cp -r $ROOT/paper_2510_11023_b200 $ROOT/include /tmp/ptrace/
cp $ROOT/tools/variants/$1.so /tmp/ptrace/paper_2510_11023_b200/libparafrac_b200.so
sed "s#/root/repo#/tmp/ptrace#" $ROOT/tools/r02/early_phase.py > /tmp/ptrace/early.py
PF_NO_HEADSTART=1 python /tmp/ptrace/early.py
