#!/bin/bash
# round-2 check 2: checksum gathers per hit + C1 bulk-copy ring variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest2.log
timeout 600 python tools/ab.py --config c4 --libs base,_c1r4,_c1r8,_c1r4m3 --flags 0,1 >> gpurun_out/ab2.jsonl 2>>gpurun_out/ab2.err
timeout 900 python tools/ab.py --config c5 --libs base,_c1r4,_c1r8 --flags 1 --reps 3 >> gpurun_out/ab2.jsonl 2>>gpurun_out/ab2.err
