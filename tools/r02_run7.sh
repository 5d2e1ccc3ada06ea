#!/bin/bash
# staged (bulk-copy ring, 4 chunks per stage) C1 / H variants; then the full-size parity suite
mkdir -p gpurun_out
timeout 900 python tools/ab.py --config c4 --libs base,_c1s2,_c1s2w17,_hcta,_hcta3 --flags 0,1 >> gpurun_out/ab7.jsonl 2>>gpurun_out/ab7.err
timeout 900 python tools/ab.py --config c5 --libs base,_hcta,_hcta3 --flags 1 --reps 2 >> gpurun_out/ab7.jsonl 2>>gpurun_out/ab7.err
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
