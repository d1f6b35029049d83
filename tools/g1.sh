set -u
O=gpurun_out/r3n; mkdir -p $O
python tools/stamps.py $O/stamps.txt > $O/stamps.log 2>&1; echo "stamps rc=$?"; cat $O/stamps.log
SGWG_P4_OVERLAP=0 python tools/stamps.py $O/stamps_noovl.txt > $O/stamps_noovl.log 2>&1; cat $O/stamps_noovl.log
