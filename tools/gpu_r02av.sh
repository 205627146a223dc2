mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged --no-e2e > gpurun_out/r02av_bench.json 2> gpurun_out/r02av_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02av_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],{x:(round(k[x]['ms']/20,2),k[x]['GB/s']) for x in ['l1_gs_f32','l1_residual_f32','l0_gs_f32','l0_residual_f64']})"
