set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ --kernel-name-base mangled -k regex:l0_hsweep_kernel.*Lb1E -c 1 -o gpurun_out/hsf -f $B > gpurun_out/hsf.log 2>&1
ncu -i gpurun_out/hsf.ncu-rep --page raw --csv > gpurun_out/hsf.raw.csv 2>/dev/null
ncu -i gpurun_out/hsf.ncu-rep --page details --csv > gpurun_out/hsf.details.csv 2>/dev/null
ncu -i gpurun_out/hsf.ncu-rep --page source --csv --print-source sass > gpurun_out/hsf.source.csv 2>/dev/null
find gpurun_out -name '*.ncu-rep' -size +20M -delete
ls -la gpurun_out
