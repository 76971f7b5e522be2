"""Warp-stall samples of an ncu report by source line range, with the stall
reasons of each (tool).  usage: ncu_regions.py report.ncu-rep file:lo-hi[=name] ..."""
import collections
import csv
import subprocess
import sys

REASONS = ["stall_long_sb", "stall_short_sb", "stall_wait", "stall_barrier", "stall_math", "stall_mio",
           "stall_lg", "stall_no_inst", "stall_branch_resolving", "stall_dispatch", "stall_not_selected",
           "stall_selected", "stall_drain", "stall_membar", "stall_misc"]


def main(rep, *specs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    rc = {k: hdr.index(k) for k in REASONS if k in hdr}
    regions = []
    for s in specs:
        f, rest = s.split(":")
        rng, _, name = rest.partition("=")
        lo, hi = (int(x) for x in rng.split("-"))
        regions.append((f, lo, hi, name or s))
    ins, smp, why = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    fname = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or not r[0] or len(r) <= ie or r[2] != "-":
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        key = next((n for f, lo, hi, n in regions if f == fname and lo <= ln <= hi), "other")
        ins[key] += int(r[ie] or 0)
        smp[key] += int(r[ws] or 0)
        for k, c in rc.items():
            why[key][k] += int(r[c] or 0)
    ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
    for k in sorted(smp, key=lambda k: -smp[k]):
        top = ", ".join(f"{a[6:]} {100 * b / max(1, smp[k]):.0f}%" for a, b in why[k].most_common(5))
        print(f"{k:24s} inst {100 * ins[k] / ti:5.1f}%  samples {100 * smp[k] / ts:5.1f}%  [{top}]")


if __name__ == "__main__":
    main(*sys.argv[1:])
