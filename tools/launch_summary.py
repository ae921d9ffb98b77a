"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

    python tools/launch_summary.py gpurun_out/launches_r01q.csv "r01q" "<cmd>" > profiles/...

Prints share %, total us, launch count per kernel name (ncu's serialised cold-cache
replays: compare shares, not absolutes).
"""

import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def main():
    path, tag, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        tot[name] += us
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none, "
          "all OUR kernels)")
    print(f"# cmd: {cmd}")
    print("# cold-cache serialised replays: compare SHARES, not absolutes; warm shares: "
          "bench.py --profile")
    print(f"# total {all_us / 1e3:.3f} ms over {sum(cnt.values())} launches")
    print("share_pct,total_us,launches,kernel")
    for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{100 * us / all_us:.1f},{us:.1f},{cnt[name]},{name}")


if __name__ == "__main__":
    main()
