# round-end validation: full GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/r02bi_gpu.log 2>&1; echo gpu rc $?
tail -3 gpurun_out/r02bi_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bi_smoke.log 2>&1; echo smoke rc $?
tail -1 gpurun_out/r02bi_smoke.log
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02bi_ref.json 2> gpurun_out/r02bi_ref.err; echo ref rc $?
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02bi_bench.json 2> gpurun_out/r02bi_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02bi_bench.json').read().strip().splitlines()[-1]);r=json.loads(open('gpurun_out/r02bi_ref.json').read().strip().splitlines()[-1])
print(d['value'],d['e2e']['value'],d['gpu_launches']/40,d['roofline']['frac'],d['clocks'],d['host_staged']['value'],d['host_staged']['hbm_library_gb'],d['reference_precision']['value'],d['cpu_baseline']['value'],r['value'])"
