# r02l: ncu --set full of one plain level-0 f32 GS colour pass (l0_gs_fast2_kernel, colour 3) at 512^3,
# with the source page for the instruction mix.
mkdir -p gpurun_out
python tools/kernel_bench.py --reso 512 --ops l0_defect_f64,l0_residual_f32 --reps 3 > gpurun_out/r02l_kb.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:hsweep -s 1 -c 1 -o gpurun_out/r02l_gs -f \
  python tools/kernel_bench.py --reso 512 --ops l0_defect_f64 --reps 1 > gpurun_out/r02l_gs.log 2>&1
ncu -i gpurun_out/r02l_gs.ncu-rep --page raw --csv > gpurun_out/r02l_gs.raw.csv 2>/dev/null
ncu -i gpurun_out/r02l_gs.ncu-rep --page source --csv > gpurun_out/r02l_gs.src.csv 2>/dev/null
gzip -f gpurun_out/r02l_gs.raw.csv gpurun_out/r02l_gs.src.csv
find gpurun_out -name '*.ncu-rep' -delete
