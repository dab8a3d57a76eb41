"""Summarise an ncu --set full capture of k_fused into profiles/ (text + JSON).

    python scripts/ncu_summarize.py gpurun_out/fused_cfg2_v5.ncu-rep cfg2 10 r01_fused

`iters` is the number of solver iterations inside the profiled launch, so that
DRAM bytes are reported per iteration (what bench.py's roofline.traffic uses).
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ncu(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, cfg, iters, tag):
    iters = int(iters)
    raw = ncu(rep, "--page", "raw", "--csv")
    hdr, units, vals = raw[0], raw[1], raw[2]
    R = dict(zip(hdr, vals))

    def f(k):
        try:
            return float(R[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    det = ncu(rep, "--page", "details", "--csv")
    dh = det[0]
    D = {}
    for row in det[1:]:
        d = dict(zip(dh, row))
        D[d.get("Metric Name")] = (d.get("Metric Value"), d.get("Metric Unit"))
    # dram__bytes_{read,write}.sum are reported in the unit row (GB / MB)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    u = dict(zip(hdr, units))
    rd = f("dram__bytes_read.sum") * scale.get(u.get("dram__bytes_read.sum"), 1)
    wr = f("dram__bytes_write.sum") * scale.get(u.get("dram__bytes_write.sum"), 1)
    dur_ms = float(D["Duration"][0]) * {"ms": 1, "us": 1e-3, "s": 1e3}[D["Duration"][1]]
    keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
            "Achieved Active Warps Per SM", "Registers Per Thread", "Dynamic Shared Memory Per Block",
            "Grid Size", "Block Size", "Executed Instructions"]
    summary = {
        "report": os.path.basename(rep), "kernel": "pf::k_fused", "config": cfg, "iterations_in_launch": iters,
        "duration_ms": dur_ms, "ms_per_iteration_under_ncu": dur_ms / iters,
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_iteration": (rd + wr) / iters,
        "details": {k: " ".join(D[k]) for k in keys if k in D},
        "stalls": {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in hdr
                   if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                   and (f(k) or 0) > 0},
        "smem_bank_conflicts_ld": f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "smem_wavefronts": f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "note": "ncu replays serialise and run cold; compare shares, not absolute times",
    }
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_{cfg}.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    agg = os.path.join(ROOT, "profiles", "ncu_summary.json")
    allj = {}
    if os.path.exists(agg):
        allj = json.load(open(agg))
    allj[cfg] = {"dram_bytes_per_iteration": summary["dram_bytes_per_iteration"], "source": f"{tag}_{cfg}.json"}
    with open(agg, "w") as fh:
        json.dump(allj, fh, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
