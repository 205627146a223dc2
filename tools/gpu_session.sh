set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_slabs.py -q 2>&1 | tail -40 > gpurun_out/slabs.log; cat gpurun_out/slabs.log
timeout 900 python -m pytest tests/ -q -m gpu -x --deselect tests/test_slabs.py 2>&1 | tail -5
