"""Summarise an ncu report (tool): stall reasons, top metrics, and warp-sample
share per SASS function (functions mapped via cuobjdump of libgevo.so)."""
import csv
import re
import subprocess
import sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main(rep, lib="paper_2310_10211_b200/libgevo.so", kernel="eval_kernel"):
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
              "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
        if k in get:
            print(f"{k:70s} {get[k][0]} {get[k][1]}")
    st = sorted(((float(v), h) for h, (v, u) in get.items()
                 if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")),
                reverse=True)[:8]
    print("stalls:", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in st))
    # SASS samples
    rows = ncu_csv(rep, "--page", "source", "--print-source=sass")
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    ie = h.index("Instructions Executed")
    sass = [(r[src].strip(), int(r[si] or 0), int(r[ie] or 0)) for r in rows[2:] if len(r) > si]
    # function boundaries from cuobjdump (same instruction order)
    dump = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = []   # (name, n_instr)
    cur, n = None, 0
    want = False
    for line in dump.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if cur:
                funcs.append((cur, n))
            cur, n = m.group(1), 0
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", line):
            n += 1
    if cur:
        funcs.append((cur, n))
    # the profiled kernel's module contains the kernel + its callees, in dump order
    tot = sum(s for _, s, _ in sass)
    print(f"total samples {tot}, sass instrs {len(sass)}")
    names = [f for f in funcs]
    # greedy: walk sass in order, assign by cumulative instr counts starting at the kernel
    idx = [i for i, (f, _) in enumerate(names) if kernel in f]
    per = Counter()
    pos = 0
    order = names[idx[0]:] + names[:idx[0]] if idx else names
    for f, cnt in order:
        per[f] += sum(s for _, s, _ in sass[pos:pos + cnt])
        pos += cnt
        if pos >= len(sass):
            break
    for f, s in per.most_common(14):
        print(f"{100 * s / max(tot, 1):5.1f}%  {f[:110]}")
    ops = Counter()
    for ins, s, _ in sass:
        t = ins.split()
        if not t:
            continue
        ops[t[1] if t[0].startswith("@") else t[0]] += s
    print("by opcode:", ", ".join(f"{k}={100 * v / max(tot, 1):.1f}%" for k, v in ops.most_common(10)))


if __name__ == "__main__":
    main(*sys.argv[1:])
