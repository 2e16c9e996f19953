"""Write profiles/<round>_summary.md + profiles/ncu_traffic.json from the ncu
artefacts of one round: the launch-list CSV (profiles/<round>_bench_launches.csv)
and `--set full` reports profiles/prof_<round>_<tag>.ncu-rep of the GEMV.

    python tools/profile_summary.py r2

Units come from the CSV unit row (tools/ncu_csv.py): round 1's version assumed
Mbyte everywhere and turned the q capture's 67.6 KB of DRAM writes into 67.6 MB.
"""
import csv
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_csv  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")

# tag -> (M, K, bits, group, k, B)
SHAPES = {
    "q": (12288, 12288, 3, 0, 15, 1), "fc1": (49152, 12288, 3, 0, 3, 1), "fc2": (12288, 49152, 3, 0, 15, 1),
    "qkv": (3 * 12288, 12288, 3, 0, 15, 1),
    "b8": (12288, 12288, 3, 0, 15, 8), "b16": (12288, 12288, 3, 0, 15, 16),
    "g128": (12288, 12288, 4, 128, 15, 1), "llama_up_b8": (11008, 4096, 4, 128, 1, 8),
    "cc_q": (12288, 12288, 3, 0, 15, 1), "cc_g128": (12288, 12288, 4, 128, 15, 1),
    "sb_llama_up_b8": (11008, 4096, 4, 128, 1, 8), "prefill": (12288, 12288, 3, 0, 15, 2048),
    "sb_llama_up_b8_v2": (11008, 4096, 4, 128, 1, 8), "prefill_v2": (12288, 12288, 3, 0, 15, 2048),
    "prefill_v3": (12288, 12288, 3, 0, 15, 2048),
    "prefill_v4": (12288, 12288, 3, 0, 15, 2048),   # one K piece (64 super-steps) of the split launch
}


def algorithmic_bytes(M, K, bits, group, k, B):
    """codes + fp16 scale/zero + weak values/indices + x + y (f16)."""
    G = 1 if group == 0 else -(-K // group)
    return bits * M * K / 8 + 4 * M * G + 2 * M * k + 2 * k + 2 * K * B + 2 * M * B


def main(rnd):
    out = [f"# ncu summary, round {rnd[1:]}\n"]
    lpath = os.path.join(P, f"{rnd}_bench_launches.csv")
    if os.path.exists(lpath):
        rows = list(csv.reader(open(lpath)))
        h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        hdr = rows[h]
        iK, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        d = defaultdict(list)
        for r in rows[h + 1:]:
            if len(r) == len(hdr):
                d[r[iK].split("(")[0]].append(float(r[iV].replace(",", "")) * ncu_csv.scale_of(r[iU]))
        tot = sum(sum(v) for v in d.values())
        out.append("## Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of "
                   "`bench.py` (cold, serialised launches)\n")
        out.append("| kernel | launches | median us | share of GPU time |\n|---|---|---|---|")
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            out.append(f"| `{k}` | {len(v)} | {sorted(v)[len(v) // 2] * 1e6:.2f} | {sum(v) / tot * 100:.1f}% |")
    traffic = {}
    out.append("\n## `ncu --set full` of one GEMV launch per shape\n")
    out.append("| shape | kernel | B | duration us | DRAM read MB | DRAM write MB | algorithmic MB | read / alg | "
               "ALU % | FMA % | tensor-mem active % | issue % | SM MHz |")
    out.append("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for tag, shp in SHAPES.items():
        rep = os.path.join(P, f"prof_{rnd}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            continue
        L = ncu_csv.launches(rep, "owq_")
        if not L:
            continue
        g = L[0]
        kname = str(g.get("Kernel Name", g.get("Function Name", "?"))).split("(")[0].split("<")[0]
        alg = algorithmic_bytes(*shp)
        rd, wr = g["dram__bytes_read.sum"], g["dram__bytes_write.sum"]
        dur = g["gpu__time_duration.sum"]

        def pct(n):
            v = g.get(n)
            return f"{v:.1f}" if isinstance(v, float) else "-"

        tc = "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"
        traffic[tag] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "algorithmic_bytes": alg,
                        "duration_us": dur * 1e6, "batch": shp[5]}
        out.append(f"| {tag} {shp[0]}x{shp[1]} b{shp[2]} g{shp[3]} k{shp[4]} | `{kname}` | {shp[5]} | {dur * 1e6:.2f} | "
                   f"{rd / 1e6:.3f} | {wr / 1e6:.4f} | {alg / 1e6:.3f} | {rd / alg:.4f} | "
                   f"{pct('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active')} | "
                   f"{pct('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active')} | "
                   f"{pct(tc) if tc else '-'} | "
                   f"{pct('sm__inst_issued.avg.pct_of_peak_sustained_active')} | "
                   f"{g.get('sm__cycles_elapsed.avg.per_second', 0) / 1e6:.0f} |")
    out.append("\n`--set full` durations are cold-cache serialised ncu replays, not bench numbers. "
               "DRAM bytes come from `dram__bytes_read.sum` / `dram__bytes_write.sum` scaled by the unit "
               "row of the CSV; `read / alg` = DRAM read over the algorithmic bytes of SURVEY §8(d).")
    open(os.path.join(P, f"{rnd}_summary.md"), "w").write("\n".join(out) + "\n")
    if traffic:
        json.dump({"round": rnd, "per_shape": traffic,
                   "note": "dram__bytes_read.sum + dram__bytes_write.sum (unit row applied) of one "
                           "--set full capture per shape"},
                  open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2")
