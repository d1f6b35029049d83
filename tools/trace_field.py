"""Phase clocks of the Vlasov-Poisson field kernel per member (experiment build
with -DSGWG_TRACE, loaded via SGWG_LIB): rho load + twiddles, forward FFT,
spectral step, inverse FFT, E store + max."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

cfg = configs.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
ctx = sgwg.Context(0, arith="fast")
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
fam.vp_field()
buf = np.zeros((128, 8), dtype=np.int64)
assert sgwg.load().sgwg_ftrace_dump(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
for mi in range(fam.num_members):
    t = buf[mi, :6].astype(np.float64)
    d = np.diff(t)
    print(f"member {mi:3d} nx={int(np.prod(fam.points[mi][:cfg['space_dim']])):5d} "
          f"load {d[0]:7.0f} fwd {d[1]:7.0f} spec {d[2]:7.0f} inv {d[3]:7.0f} out {d[4]:7.0f} "
          f"total {t[5]-t[0]:8.0f}")
