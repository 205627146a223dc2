mkdir -p gpurun_out
cap() {  # tag regex skip op
  timeout 400 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$2 -s $3 -c 1 \
    -o gpurun_out/r02u_$1 -f python tools/kernel_bench.py --reso 512 --ops $4 --reps 1 > gpurun_out/r02u_$1.log 2>&1
  ncu -i gpurun_out/r02u_$1.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02u_$1.raw.csv.gz
  ncu -i gpurun_out/r02u_$1.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/r02u_$1.src.csv.gz
  rm -f gpurun_out/r02u_$1.ncu-rep
}
cap gal gal_stencil_fast_kernel 6 set_density
cap gs l0_gs_fast2_kernelIffLi5ELb0ELin1E 10 l0_gs_f32
du -sh gpurun_out
