# one GPU round trip: parity tests, smoke, bench, reference arm, ncu launch
# list + one full capture of eval_kernel (-> profiles/traffic.json via
# tests/tools/ncu_traffic.py, stamped with the sha of the library profiled)
# usage: bash tests/tools/gpu_run.sh [tag] [bench args...]
TAG=${1:-run}; shift
BENCH_ARGS=${@:---steps 5 --warmup 3}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${TAG}_tests.log 2>&1
grep -E "bit-exact|passed|failed|Error|error" gpurun_out/${TAG}_tests.log | tail -14
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; tail -n 1 gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py $BENCH_ARGS > gpurun_out/${TAG}_bench.log 2>&1; tail -n 2 gpurun_out/${TAG}_bench.log
if [ -z "$NO_REF" ]; then
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference_arm.log 2>&1; tail -n 1 gpurun_out/${TAG}_reference_arm.log
fi
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cnn --no-e2e --no-tf32 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/${TAG}_prof python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cnn --no-e2e --no-tf32 > gpurun_out/${TAG}_ncu.log 2>&1
tail -n 1 gpurun_out/${TAG}_ncu.log
fi
