"""Median per-iteration timeline of a multi-GPU solve traced with
SBX_TRACE=<prefix> (one file per rank: <prefix>.rank<r>).

    python tools/trace_summary.py gpurun_out/trace
"""
import glob
import statistics
import sys

SEG = [("K1 head: r'z/r'r exchange + step", 0, 6), ("K1 body (-> last CTA)", 6, 1),
       ("K1 end -> K2 start", 1, 2), ("K2: release + wait for peers", 2, 3),
       ("interface groups + grid barrier", 3, 4), ("K2 body (-> last CTA)", 4, 5),
       ("K2 last CTA -> next K1 start", 5, 7)]
SEG1 = [("K1 (CTA0 start -> last CTA)", 0, 1), ("K1 end -> K2 start", 1, 4),
        ("K2 body (-> last CTA)", 4, 5), ("K2 last CTA -> next K1 start", 5, 8)]


def main(prefix):
    for path in sorted(glob.glob(prefix + ".rank*")):
        rows = [list(map(int, l.split())) for l in open(path)]
        rows.sort()
        its = {r[0]: r[1:] for r in rows}
        # single GPU (SBX_TRACE1): slots 2, 3, 6 are not stamped
        single = all(r[3] == 0 and r[4] == 0 for r in its.values())
        seg = SEG1 if single else SEG
        acc = {name: [] for name, _, _ in seg}
        tot = []
        for it, t in its.items():
            if it < 3 or it + 1 not in its:
                continue
            nxt = its[it + 1][0]
            t = t + [nxt]
            if min(t[a] for _, a, b in seg) == 0 or min(t[b] for _, a, b in seg) == 0:
                continue
            for name, a, b in seg:
                acc[name].append((t[b] - t[a]) / 1e3)
            tot.append((nxt - t[0]) / 1e3)
        print(f"{path}: {len(tot)} iterations, median {statistics.median(tot):.1f} us/iteration")
        for name, _, _ in seg:
            print(f"  {name:32s} {statistics.median(acc[name]):8.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
