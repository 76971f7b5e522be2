timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/r02i_tests.log 2>&1; tail -3 gpurun_out/r02i_tests.log
grep -E "bit-exact|mismatch|replay" gpurun_out/r02i_tests.log | tail -12
timeout 300 python __graft_entry__.py > gpurun_out/r02i_smoke.log 2>&1; tail -n 1 gpurun_out/r02i_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02i_bench.log 2>&1; tail -n 1 gpurun_out/r02i_bench.log | cut -c1-1500
