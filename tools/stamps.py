"""Timeline of a captured C5 step from the SGWG_STAMPS device-clock stamps
(timing experiments only): medians of the segment lengths over the steps of the
first 64-step graph's last replay."""
import os, sys, statistics as st
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/stamps.txt"
os.environ["SGWG_STAMPS"] = out
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

cfg = configs.config("C5")
ctx = sgwg.Context(0, arith="fast")
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
dts = fam.evolve_config(cfg, tfinal=0.52, stops=[])
s = fam.stats()
print("steps", len(dts), "evolve_ms", s.get("evolve_ms"), "us/step", 1e3 * s.get("evolve_ms", 0) / max(1, len(dts)))
rows = [tuple(map(int, l.split())) for l in open(out)]
# split into steps at label 0
steps, cur = [], None
for lab, t in rows:
    if lab == 0:
        cur = {}
        steps.append(cur)
    if cur is not None:
        cur[lab] = t
steps = [x for x in steps[:64] if all(v > 0 for v in x.values())]
def med(f):
    v = [f(x) for x in steps if f(x) is not None]
    return st.median(v) / 1e3 if v else float("nan")
def d(a, b):
    return lambda x: (x[b] - x[a]) if a in x and b in x else None
print("steps with stamps", len(steps))
for name, a, b in [("field1 (0->31)", 0, 31), ("dt (31->1)", 31, 1), ("xpass1 end after dt (1->21)", 1, 21),
                   ("energy end after dt (1->11)", 1, 11),
                   ("join1 (1->41)", 1, 41), ("vpass1 (41->51)", 41, 51), ("field2 (51->32)", 51, 32),
                   ("xpass2 end after field2 (32->22)", 32, 22), ("join2 (32->42)", 32, 42),
                   ("vpass2 (42->52)", 42, 52), ("field3 (52->33)", 52, 33),
                   ("xpass3 end after field3 (33->23)", 33, 23), ("join3 (33->43)", 33, 43),
                   ("vpass3 (43->53)", 43, 53), ("step (0->53)", 0, 53),
                   ("stage1 x+v (0->51)", 0, 51), ("stage2 (51->52)", 51, 52), ("stage3 (52->53)", 52, 53)]:
    print(f"{name:40s} {med(d(a, b)):9.1f} us")
nxt = [steps[i + 1][0] - steps[i][53] for i in range(len(steps) - 1) if 53 in steps[i]]
if nxt:
    print(f"{'step end -> next step start':40s} {st.median(nxt) / 1e3:9.1f} us")
