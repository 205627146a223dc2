# r02d: kernel bench + ncu --set full of the f64 modal tensor pass (256^3) and its f32 twin.
mkdir -p gpurun_out
python tools/kernel_bench.py --reso 256 --ops tensor,sensitivity --reps 3 > gpurun_out/r02f_kb.json 2>&1
IHOM_ENERGY_F32=1 python tools/kernel_bench.py --reso 256 --ops tensor --reps 3 >> gpurun_out/r02f_kb.json 2>&1
full() {  # name regex count [env]
  timeout 900 env $4 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$2 -c $3 \
    -o gpurun_out/r02f_$1 -f python tools/kernel_bench.py --reso 256 --ops tensor --reps 1 > gpurun_out/r02f_$1.log 2>&1
  ncu -i gpurun_out/r02f_$1.ncu-rep --page raw --csv > gpurun_out/r02f_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/r02f_$1.ncu-rep --page source --csv > gpurun_out/r02f_$1.src.csv 2>/dev/null
  gzip -f gpurun_out/r02f_$1.raw.csv gpurun_out/r02f_$1.src.csv
}
full tensor_stage 'tensor_stage_kernel' 1

find gpurun_out -name '*.ncu-rep' -delete
