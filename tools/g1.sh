set -u
O=gpurun_out/r3d; mkdir -p $O
python tools/energy_ab.py > $O/energy_ab.log 2>&1; cat $O/energy_ab.log
python tools/stamps.py $O/stamps.txt > $O/stamps.log 2>&1; echo "stamps rc=$?"; cat $O/stamps.log
python tools/profile_evolve.py --config C5 --tfinal 0.52 > $O/plain.log 2>&1; cat $O/plain.log
