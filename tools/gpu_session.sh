# z-slab bring-up: slab tests first (short timeout: a collective mismatch would hang), then the GPU suite
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_slabs.py -x -q 2>&1 | tail -30 > gpurun_out/slabs.log; cat gpurun_out/slabs.log
timeout 900 python -m pytest tests/ -q -m gpu -x --deselect tests/test_slabs.py 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline --steps 2 > gpurun_out/bench512_slabbuild.json 2> gpurun_out/bench512_slabbuild.err; tail -2 gpurun_out/bench512_slabbuild.err
