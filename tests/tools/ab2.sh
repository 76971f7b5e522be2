# ABAB: bench (MLP value + CNN) with the main library and an alternative build
ALT=$1
cp paper_2310_10211_b200/libgevo.so /tmp/libgevo_main.so
for r in 1 2; do
  for lib in /tmp/libgevo_main.so $ALT; do
    cp $lib paper_2310_10211_b200/libgevo.so
    timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 > gpurun_out/ab_bench.log 2>&1
    echo "$lib $(python -c "import json;l=json.loads(open('gpurun_out/ab_bench.log').read().strip().splitlines()[-1]);print('mlp', round(l['value'],1), 'cnn', round(l['cnn']['value'],2))" 2>&1 | tail -1)"
  done
done
cp /tmp/libgevo_main.so paper_2310_10211_b200/libgevo.so
