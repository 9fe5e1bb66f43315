#!/bin/bash
# Whole GPU check of the current build (run under gpurun): GPU test suite, smoke(), default bench line.
set -o pipefail
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv | tee gpurun_out/full_gpuinfo.txt
python -m pytest tests/ -q -m gpu --durations=25 2>&1 | tee gpurun_out/full_pytest.log | tail -40
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -3 | tee gpurun_out/full_smoke.log
python bench.py 2>gpurun_out/full_bench.err | tee gpurun_out/full_bench.json | tail -1 | cut -c1-600
