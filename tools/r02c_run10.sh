#!/bin/bash
# class-H split (warp kernel for small sets on large graphs): A/B on C5; wide paths at C4
mkdir -p gpurun_out
A="timeout 900 python tools/ab.py --class-work --reps 2"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wide_h or cli" > gpurun_out/c11_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c11_pytest.log
$A --config c5 --libs _hs --flags 1 --hsplit 0,48,64,96,128,256 >> gpurun_out/c11_ab.jsonl 2>>gpurun_out/c11_ab.err
$A --config c4 --libs _hs --flags 1 --hwide-min-n 0 --hsplit 0,64,256 >> gpurun_out/c11_ab.jsonl 2>>gpurun_out/c11_ab.err
echo done
