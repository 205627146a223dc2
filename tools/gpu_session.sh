set -x
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mbp tools/microbench_pipes.cu && /tmp/mbp > gpurun_out/pipes.txt 2>&1
for k in l0_gs_fast2_kernel l0_residual_norm_fast_kernel l0_apply_fast_kernel; do
  op=l0_gs_f32; [ $k = l0_residual_norm_fast_kernel ] && op=l0_defect_f64; [ $k = l0_apply_fast_kernel ] && op=l0_residual_f32
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 -o gpurun_out/ncu_$k -f python tools/kernel_bench.py --reso 512 --ops $op --reps 1 > gpurun_out/ncu_$k.log 2>&1
done
