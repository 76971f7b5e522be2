# quick GPU check (tool): parity tests, dot micro-bench, op profile, short bench
TAG=${1:-q}
timeout 600 python -m pytest tests -m gpu -x -q -s > gpurun_out/${TAG}_tests.log 2>&1
grep -E "bit-exact|passed|failed|Error|error" gpurun_out/${TAG}_tests.log | tail -12
for k in small big bigsgd; do timeout 120 python tests/tools/dot_bench.py $k; done > gpurun_out/${TAG}_dot.txt 2>&1
timeout 300 python tests/tools/op_profile.py > gpurun_out/${TAG}_op.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; tail -n 1 gpurun_out/${TAG}_bench.log | cut -c1-400
