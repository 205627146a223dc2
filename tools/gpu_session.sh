# round-1 profiling session: bench with/without the family profiler, ncu launch list of the
# timed region, ncu --set full captures of the top kernels at 512^3.
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench512_prof.json 2> gpurun_out/bench512_prof.err
timeout 600 python bench.py --no-cpu-baseline --no-profile > gpurun_out/bench512_noprof.json 2>> gpurun_out/bench512_prof.err
tail -3 gpurun_out/bench512_prof.err
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches512.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile \
  > gpurun_out/launches512.log 2>&1; tail -3 gpurun_out/launches512.log
for k in l0_gs_fast2_kernel l0_residual_norm_fast_kernel stencil_gs_fast_kernel tensor_kernel sens_kernel gal_elem_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:$k -c 1 \
    -o gpurun_out/full512_$k python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile \
    > gpurun_out/full512_$k.log 2>&1; tail -2 gpurun_out/full512_$k.log
done
ls -la gpurun_out
