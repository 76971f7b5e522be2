bash tests/tools/gpu_run.sh r02f --steps 5 --warmup 3
GEVO_B200_DTYPE=tf32 timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:eval_kernel_tc -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cnn --no-e2e --no-tf32 > gpurun_out/r02f_ncu_tf32.txt 2>&1
grep -E "tensor|utchmma|duration|dram" gpurun_out/r02f_ncu_tf32.txt
timeout 900 python tests/tools/ga_bench.py > gpurun_out/r02f_ga512x50.json 2>/dev/null; tail -1 gpurun_out/r02f_ga512x50.json | cut -c1-300
timeout 900 python -c "
import sys, json; sys.path[:0]=['.', 'tests']
import bench
print(json.dumps(bench.cnn_measure(0, steps=1, n_img=10000)))" > gpurun_out/r02f_cnn10k.json 2>/dev/null; tail -1 gpurun_out/r02f_cnn10k.json
