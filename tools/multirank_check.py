"""Two-or-more-rank check of libsgwg's sharded path (one process per GPU, torchrun):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/multirank_check.py [C2|C5]

Every rank: its LPT shard (paper_2007_10196_b200/shard.py) with an NCCL communicator,
the evolve (per-step all-reduce(max) of the wave speeds), then option B: sgwg_combine_local
(this rank's dimension-0 rows, every member gathered), combined_stats and a cut plane.
Rank 0 also runs the unsharded family on its GPU; every rank's rows must be BITWISE the
unsharded combination's rows, the dt sequences and the cut plane bitwise equal, the stats
within 1e-13.  Finally a non-finite state injected into one member owned by the last rank
must make EVERY rank raise FamilyIntegratorFailure with the same (member, step, stage).
Prints one JSON line per rank; exit code 0 = all checks passed."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2007_10196_b200 import configs, sgwg, shard  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
over = {"C2": {"nl": 4, "root": [16, 16]}, "C5": {"nl": 3}}.get(name, {})
T = {"C2": 0.05, "C5": 0.05}.get(name, 0.02)
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = configs.config(name, **over)
ctx = sgwg.Context(local, arith="fast")
import bench  # noqa: E402  (level enumeration without a GPU)
levels = bench._levels(cfg)
pts = shard.member_points(levels, cfg["root"], cfg["bc"])
shards = shard.lpt_shards(pts, world)
fam = sgwg.Family.from_config(ctx, cfg, members=shards[rank])
uid = [sgwg.nccl_unique_id() if rank == 0 else bytes(128)]
dist.broadcast_object_list(uid, src=0)
fam.set_comm(uid[0], world, rank)
fam.initialize(cfg["ic"])
dts = fam.evolve_config(cfg, tfinal=T, stops=[])
a, b, rows = fam.combine_local(cfg["interp"], cfg["epsilon"])
st = fam.combined_stats(cfg["interp"], cfg["epsilon"])
plane = fam.cut_plane(0, cfg["d"] - 1, [0] * cfg["d"], cfg["interp"], cfg["epsilon"])
out = {"rank": rank, "rows": [a, b], "steps": len(dts)}
ok = True
ref = None
if rank == 0:
    rfam = sgwg.Family.from_config(ctx, cfg)
    rfam.initialize(cfg["ic"])
    rdts = rfam.evolve_config(cfg, tfinal=T, stops=[])
    full = rfam.combine(cfg["interp"], cfg["epsilon"])
    rst = rfam.combined_stats(cfg["interp"], cfg["epsilon"])
    rplane = rfam.cut_plane(0, cfg["d"] - 1, [0] * cfg["d"], cfg["interp"], cfg["epsilon"])
    ref = {"dts": rdts, "full": full, "stats": rst, "plane": rplane}
    rfam.close()
gathered = [None] * world
dist.all_gather_object(gathered, (a, b, rows))
if rank == 0:
    per_row = full.size // fam.fine_extent0
    for ga, gb, grows in gathered:
        eq = np.array_equal(grows, full[ga * per_row:gb * per_row])
        out.setdefault("rows_bitwise", []).append(bool(eq))
        ok &= eq
    out["rows_cover"] = sorted(g[:2] for g in gathered)[0][0] == 0
    out["dts_bitwise"] = bool(np.array_equal(dts, ref["dts"]))
    out["plane_bitwise"] = bool(np.array_equal(plane, ref["plane"]))
    srel = max(abs(st[k] - ref["stats"][k]) / max(1.0, abs(ref["stats"][k]))
               for k in ("mass", "min", "max"))
    out["stats_rel"] = srel
    ok &= out["dts_bitwise"] and out["plane_bitwise"] and srel < 1e-13
# failure propagation: a NaN in the last rank's first member
s = fam.download()
if rank == world - 1:
    s[0] = np.nan
fam.upload(s)
try:
    fam.evolve_config(cfg, tfinal=T, stops=[])
    fail = None
except sgwg.FamilyIntegratorFailure as e:
    fail = (e.level, e.step, e.stage)
fails = [None] * world
dist.all_gather_object(fails, fail)
out["failure"] = fail
out["failure_same_on_all_ranks"] = fail is not None and all(f == fail for f in fails)
ok &= out["failure_same_on_all_ranks"]
out["ok"] = bool(ok)
print(json.dumps(out), flush=True)
fam.close()
ctx.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
