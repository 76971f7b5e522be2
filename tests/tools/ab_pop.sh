# A/B of library builds at several population sizes (tool):
# usage: bash tests/tools/ab_pop.sh "<pop list>" alt1.so [alt2.so ...]
POPS=$1; shift
cp paper_2310_10211_b200/libgevo.so /tmp/libgevo_main.so
for lib in /tmp/libgevo_main.so "$@"; do
  cp $lib paper_2310_10211_b200/libgevo.so
  for p in $POPS; do
    timeout 600 python bench.py --pop $p --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 --no-cnn > gpurun_out/ab_pop.log 2>&1
    echo "$lib pop $p $(python -c "import json;l=json.loads(open('gpurun_out/ab_pop.log').read().strip().splitlines()[-1]);print('value', round(l['value'],1), 'ms', round(l['ms_per_step'],1), 'parity', l['parity']['bit_exact'], '/', l['parity']['of'])" 2>&1 | tail -1)"
  done
done
cp /tmp/libgevo_main.so paper_2310_10211_b200/libgevo.so
