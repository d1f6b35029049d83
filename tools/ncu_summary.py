"""Summarise ncu reports (gpurun_out/*.ncu-rep) into compact JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] > profiles/<round>_<name>.json

Per profiled launch: duration, SM-active vs elapsed cycles, fp64-pipe and
issue utilisation, DRAM bytes (traffic), occupancy, registers, instruction
mix (DFMA/DMUL/DADD), top warp-stall reasons.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_us",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
    "sm__cycles_active.avg": "sm_active_cycles_avg",
    "sm__cycles_active.max": "sm_active_cycles_max",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_pct_active",
    "smsp__inst_executed.sum": "warp_instructions",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "thread_dfma",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "thread_dmul",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "thread_dadd",
}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        stalls = {}
        for i, h in enumerate(hdr):
            v = r[i].replace(",", "")
            try:
                fv = float(v)
            except ValueError:
                continue
            if h in WANT:
                key = WANT[h]
                u = units[i]
                if key.startswith("dram_") and u:  # normalise to bytes
                    fv *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if key == "duration_us" and u == "nsecond":
                    fv /= 1e3
                if key == "duration_us" and u == "msecond":
                    fv *= 1e3
                d[key] = fv
            elif h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = fv
        if stalls:
            tot = sum(stalls.values()) or 1.0
            d["stall_share"] = {k: round(v / tot, 3) for k, v in
                                sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        if "dram_read" in d and "dram_write" in d:
            d["traffic_bytes"] = d["dram_read"] + d["dram_write"]
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps({p: raw(p) for p in sys.argv[1:]}, indent=1))
