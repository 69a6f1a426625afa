#!/bin/bash
# r03z: sanity after the device_bytes accounting change: parity tests, smoke, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-400
