"""Per-source-line instruction and warp-sample shares of an ncu report (tool)."""
import collections
import csv
import subprocess
import sys


def main(rep, n=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    fname = None
    ins, smp = collections.Counter(), collections.Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or not r[0] or len(r) <= ie or r[2] != "-":
            continue
        try:
            k = (fname, int(r[0]), r[1].strip()[:80])
            ins[k] += int(r[ie] or 0)
            smp[k] += int(r[ws] or 0)
        except ValueError:
            continue
    ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
    keys = sorted(set(ins) | set(smp), key=lambda k: -(ins[k] / ti + smp[k] / ts))
    for k in keys[:int(n)]:
        print(f"{100 * ins[k] / ti:5.1f}% inst {100 * smp[k] / ts:5.1f}% smp  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
