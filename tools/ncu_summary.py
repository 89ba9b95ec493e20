#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, total device time, share.  Usage: ncu_summary.py launches.csv [--window MARKER]
--window: only the launches from the first launch whose name contains MARKER up to (not
including) the next one -- e.g. xent_pipe_kernel, once per training step."""
import csv
import collections
import re
import sys


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    if "--window" in sys.argv:
        # MARKER[:N]: from the first launch whose name contains MARKER to its N-th next occurrence
        # (N = launches of MARKER per step, e.g. 2 head-loss launches per CheckFree+ step)
        mk = sys.argv[sys.argv.index("--window") + 1]
        n = 1
        if ":" in mk:
            mk, n = mk.rsplit(":", 1)
            n = int(n)
        idx = [i for i, r in enumerate(rows) if mk in r[4]]
        if len(idx) >= n + 1:
            rows = rows[idx[0]:idx[n]]
    tot = collections.OrderedDict()
    for r in rows:
        name = re.sub(r"\(.*", "", r[4]).replace("void ", "")
        ns = float(r[-1].replace(",", ""))
        t = tot.setdefault(name, [0, 0.0])
        t[0] += 1
        t[1] += ns
    all_ns = sum(v[1] for v in tot.values())
    print(f"{len(rows)} launches, {all_ns / 1e6:.3f} ms total (cold-cache, serialised ncu replay)")
    print(f"{'kernel':<90} {'n':>6} {'ms':>10} {'share':>7}")
    for k, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:90]:<90} {n:>6} {ns / 1e6:>10.3f} {ns / all_ns:>7.1%}")


if __name__ == "__main__":
    main()
