# BASELINE.json configs[4] at N=1: population sweep of the bench workload
# (train2fc, distinct recorded GA variants, cycled when P > pool size).
# usage: bash tests/tools/pop_sweep.sh [out.jsonl]
OUT=${1:-gpurun_out/pop_sweep.jsonl}
: > $OUT
for P in 64 128 256 512 1024 2048 4096; do
  timeout 900 python bench.py --pop $P --steps 3 --warmup 3 --no-cpu-baseline --no-cnn --no-tf32 | tail -n 1 >> $OUT
  python - "$OUT" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().splitlines()[-1])
print(l["config"]["population_per_gpu"], round(l["value"], 1), round(l["e2e"]["value"], 1),
      round(l["ms_per_step"], 2), l["parity"])
PY
done
