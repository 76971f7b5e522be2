# bf16 tcgen05 mode: the tc tests for both modes, then the f64 gate and one
# bench line per mode (device rate of the population)
timeout 900 python -m pytest tests/test_tc.py -x -q -s 2>&1 | grep -E "dots:|train_step:|exact|passed|failed|Error" | tail -12
for d in f64 tf32 bf16; do
GEVO_B200_DTYPE=$d timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cnn --no-e2e --no-tf32 2>/dev/null | tail -n 1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$d', round(j['value'],1), j['ms_per_step'])"
done
