timeout 900 python -c "
import sys, json; sys.path[:0]=['.', 'tests']
import bench
print(json.dumps(bench.cnn_measure(0, steps=1, n_img=10000)))" > gpurun_out/r02_cnn10k.json 2>gpurun_out/r02_cnn10k.err; tail -1 gpurun_out/r02_cnn10k.json
timeout 900 python tests/tools/ga_bench.py > gpurun_out/r02_ga512x50.json 2>gpurun_out/r02_ga.err; tail -1 gpurun_out/r02_ga512x50.json
