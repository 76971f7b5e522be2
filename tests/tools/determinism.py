"""Run the same 256-individual plan 4 times (tool): results must match each
other and the reference; GEVO_POISON=1 fills the arena with NaN first, so a
read of memory no instruction wrote shows up as a mismatch."""
import sys
sys.path[:0]=['/root/repo','/root/repo/tests']
import numpy as np
from golden_io import load
from paper_2310_10211_b200.dialect import parse_function
from paper_2310_10211_b200 import workloads as W
from paper_2310_10211_b200.evaluator import DeviceEvaluator, lower_all
from paper_2310_10211_b200.plan import build_population_plan
inds=load("bench_train_pool.json.gz")["individuals"]
seen=set(); pool=[]
for i in inds:
    if i["key"] not in seen: seen.add(i["key"]); pool.append(i)
wl=W.build_2fcnet_workload(); ev=DeviceEvaluator(wl)
V=[{n: parse_function(i[n]) for n in ("forward","train_step")} for i in pool[:256]]
vps=lower_all(V, None, True)
p=build_population_plan(vps, ev.weight_shapes, 320)
outs=[]
for t in range(4):
    res,_=ev.ctx.eval(p.blob, p.n_prog, 0, 600, 50, 0, 0, ev.weight_elems, False)
    outs.append(res[["wrong","status"]].copy())
    bad=[(k, int(r["wrong"]), int(r["status"])) for k,r in enumerate(res) if (r["status"]!=0)!=(pool[k]["error"]==1.0) or (r["status"]==0 and r["wrong"]/992 != pool[k]["error"])]
    print("run", t, "mismatch vs reference:", bad[:8])
for t in range(1,4):
    d=np.flatnonzero(outs[t]!=outs[0])
    print("run", t, "differs from run 0 at", d[:10].tolist())
