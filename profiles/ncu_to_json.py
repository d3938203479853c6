#!/usr/bin/env python3
"""Record one ncu capture of a bench launch into profiles/ncu_bench_launch.json (read by bench.py's roofline block).

    python profiles/ncu_to_json.py <report.ncu-rep> <key> <scenarios> <requests> <summary.txt>

<key> is the kernel mode ("slots", "blocks", "c5_blocks" ...).  Per launch: DRAM bytes (traffic), duration, SM
cycles, warp instructions, issue-active %, threads per warp instruction (warp-execution efficiency), shared-memory
wavefronts and bank conflicts; per selection where it makes sense.
"""
import csv
import io
import json
import os
import subprocess
import sys

M = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "threads_per_warp_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "warp_instructions": "smsp__inst_executed.sum",
    "sm_cycles": "sm__cycles_elapsed.avg",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "ns": 1e-6}


def main():
    rep, key, S, R, summary = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, r = rows[0], rows[1], rows[2]
    out = {"scenarios": S, "requests": R, "selections": S * R, "summary": summary,
           "kernel": r[hdr.index("Kernel Name")]}
    for k, m in M.items():
        i = hdr.index(m)
        v = float(r[i].replace(",", ""))
        out[k] = v * SCALE.get(units[i], 1.0)
    out["traffic_bytes"] = out.pop("dram_read") + out.pop("dram_write")
    sel = S * R
    out["per_selection"] = {"dram_bytes": out["traffic_bytes"] / sel,
                            "warp_instructions": out["warp_instructions"] / sel,
                            "smem_wavefronts": out["smem_wavefronts"] / sel,
                            "smem_bank_conflicts": out["smem_bank_conflicts"] / sel}
    out["warp_execution_efficiency"] = out["threads_per_warp_inst"] / 32.0
    out["smem_wavefronts_per_sm_cycle"] = out["smem_wavefronts"] / (out["sm_cycles"] * 148)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_bench_launch.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[key] = out
    with open(path, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
