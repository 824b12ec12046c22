"""Summarise gpurun_out/sweep.jsonl (tools/sweep.sh) into a markdown table.

    python tools/sweep_summary.py gpurun_out/sweep.jsonl profiles/r01_scaling.md
"""
import json
import sys
from collections import defaultdict


def main(src, dst):
    rows = [json.loads(l) for l in open(src) if l.strip()]
    ok = [r for r in rows if "failed" not in r]
    by = defaultdict(dict)
    for r in ok:
        c = r["config"]
        e = tuple(c["elements"])
        by[(c["degree"], e)][r["n_gpus"]] = r
    out = ["# Strong scaling and size sweep (bench.py lines from `tools/sweep.sh`)", "",
           "GDOF/s = E·(N+1)³·iterations/s over all ranks (device-resident, max over ranks);",
           "efficiency = value / (n_gpus × 1-GPU value of the same mesh). Timing-mode K1 / K2",
           "are rank 0's per-launch averages (K2 on >1 GPU includes the halo assembly and the",
           "scalar exchange).", "",
           "| N | mesh | elements/GPU | GPUs | GDOF/s | efficiency | µs/iteration | K1 µs | K2 µs | SM MHz |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for (N, e), d in sorted(by.items(), key=lambda kv: (kv[0][0], kv[0][1])):
        base = d.get(1, {}).get("value")
        for g in sorted(d):
            r = d[g]
            E = e[0] * e[1] * e[2]
            eff = f"{r['value'] / (g * base):.2f}" if base else "–"
            rl = r.get("roofline", {})
            out.append(f"| {N} | {e[0]}×{e[1]}×{e[2]} | {E // g} | {g} | {r['value']:.1f} | {eff} | "
                       f"{r['ms_per_iteration'] * 1e3:.1f} | {rl.get('k1_ms', 0) * 1e3:.1f} | "
                       f"{rl.get('k2_ms', 0) * 1e3:.1f} | {r.get('clocks', {}).get('sm_mhz')} |")
    bad = [r for r in rows if "failed" in r]
    if bad:
        out += ["", "Failed runs: " + ", ".join(r["failed"] for r in bad)]
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
