# ncu of the plain colour-pair GS launch (kernel_bench, 512^3)
mkdir -p gpurun_out
timeout 500 ncu --set full --clock-control none --kernel-name-base mangled -k regex:l0_gs_pair_kernelIffLb0ELin1E -c 1 -o gpurun_out/r02ba_pair -f python tools/kernel_bench.py --reso 512 --ops l0_gs_f32 --reps 1 > gpurun_out/r02ba.log 2>&1; echo ncu rc $?
ncu -i gpurun_out/r02ba_pair.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02ba_pair.raw.csv.gz
rm -f gpurun_out/*.ncu-rep
