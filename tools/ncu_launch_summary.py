"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares of the profiled step.

    python tools/ncu_launch_summary.py launches.csv [out.json]

ncu times are cold-cache and serialised: compare SHARES with bench.py's
per-kernel CUDA-event table, not absolutes.
"""
import csv
import json
import re
import sys
from collections import defaultdict


def main(path, out=None):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        name = re.sub(r"^void ", "", name)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        tot[name] += v * scale
        cnt[name] += 1
    total = sum(tot.values())
    rows = sorted(tot, key=lambda k: -tot[k])
    res = {"total_ms": total, "launches": sum(cnt.values()),
           "kernels": {k: {"ms": tot[k], "launches": cnt[k], "share": tot[k] / total if total else 0}
                       for k in rows}}
    for k in rows:
        print(f"{tot[k]:12.2f} ms {cnt[k]:8d} launches {100 * tot[k] / total:6.2f}%  {k}")
    print(f"total {total:.1f} ms over {res['launches']} launches")
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
