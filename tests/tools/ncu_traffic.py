"""Record the hot kernel's DRAM traffic and pipe counters from one `ncu --set
full` capture into profiles/traffic.json, stamped with the source sha of the
build that was profiled (build.source_sha: sources + nvcc flags).  bench.py
reports `roofline.traffic` only when that sha matches the build it is running
(a capture of another build reads as null, never as a stale number).

    python tests/tools/ncu_traffic.py gpurun_out/<tag>_prof.ncu-rep <tag> [lib_sha]
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        launches.append({h: (v, u) for h, u, v in zip(hdr, units, vals)})
    return launches


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def main(rep, tag, sha=None):
    if sha is None:
        sys.path.insert(0, ROOT)
        from paper_2310_10211_b200 import build
        sha = build.source_sha()
    launches = raw_metrics(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    out = []
    for m in launches:
        rd, ru = m.get("dram__bytes_read.sum", (None, "byte"))
        wr, wu = m.get("dram__bytes_write.sum", (None, "byte"))
        dram = num(rd) * scale.get(ru, 1) + num(wr) * scale.get(wu, 1)
        pipes = {k: num(v) for k, (v, u) in m.items()
                 if ("pipe_fp64" in k or "dmma" in k or "pipe_tensor" in k)
                 and k.endswith("pct_of_peak_sustained_active")}
        out.append({"kernel": m.get("Kernel Name", ("?", ""))[0],
                    "duration_ns": num(m.get("gpu__time_duration.sum", (0, ""))[0]),
                    "dram_bytes": dram,
                    "warps_active_pct": num(m.get("sm__warps_active.avg.pct_of_peak_sustained_active",
                                                  (None, ""))[0]),
                    "pipes_pct": pipes})
    rec = {"lib_sha": sha, "source": f"profiles/{tag}_ncu_summary.md ({os.path.basename(rep)})",
           "dram_bytes_per_launch": sum(o["dram_bytes"] for o in out) / max(1, len(out)),
           "launches": out}
    path = os.path.join(ROOT, "profiles", "traffic.json")
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
