set -u
O=gpurun_out/r2g; mkdir -p $O
L=paper_2007_10196_b200
export SGWG_P4_PERSIST=0
timeout 300 python tools/profile_c5.py C5 0.02 > $O/base.json 2>&1; echo "base rc=$?"
SGWG_P4_XTARGET=2048 timeout 300 python tools/profile_c5.py C5 0.02 > $O/base_xt2048.json 2>&1; echo "rc=$?"
SGWG_LIB=$L/libsgwg_v192.so SGWG_P4_VTARGET=1800 SGWG_P4_XTARGET=3072 timeout 300 python tools/profile_c5.py C5 0.02 > $O/v192.json 2>&1; echo "v192 rc=$?"
SGWG_LIB=$L/libsgwg_v192.so SGWG_P4_VTARGET=1800 SGWG_P4_XTARGET=2048 timeout 300 python tools/profile_c5.py C5 0.02 > $O/v192_xt2048.json 2>&1; echo "v192 rc=$?"
SGWG_LIB=$L/libsgwg_v128.so SGWG_P4_VTARGET=1350 SGWG_P4_XTARGET=2048 timeout 300 python tools/profile_c5.py C5 0.02 > $O/v128.json 2>&1; echo "v128 rc=$?"
SGWG_LIB=$L/libsgwg_v128.so SGWG_P4_VTARGET=1350 SGWG_P4_XTARGET=1024 timeout 300 python tools/profile_c5.py C5 0.02 > $O/v128_xt1024.json 2>&1; echo "v128 rc=$?"
