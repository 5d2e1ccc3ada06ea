#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled" > gpurun_out/c15_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c15_pytest.log
timeout 1500 python tools/core_time.py c2 c4 c5 > gpurun_out/c15_core.jsonl 2> gpurun_out/c15_core.err
echo done
