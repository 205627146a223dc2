# final bench, both arms, as the driver runs them
mkdir -p gpurun_out
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ao_ref.json 2> gpurun_out/r02ao_ref.err; echo ref rc $?
tail -c 800 gpurun_out/r02ao_ref.json
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ao_bench.json 2> gpurun_out/r02ao_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ao_bench.json').read().strip().splitlines()[-1])
print(d['value'],d['e2e'],d['gpu_launches'],d['roofline'],d['clocks'],d.get('host_staged'),d.get('reference_precision',{}).get('value'),d.get('cpu_baseline'))"
tail -3 gpurun_out/r02ao_bench.err
