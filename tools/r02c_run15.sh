#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "scaled or shrunk or golden or sweep or c1 or edge or wide" > gpurun_out/c17_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c17_pytest.log
A="timeout 900 python tools/ab.py --class-work --reps 3"
$A --config c3 --libs base,_rs0 --flags 0,1,3 >> gpurun_out/c17_ab.jsonl 2>>gpurun_out/c17_ab.err
$A --config c2 --libs base,_rs0 --flags 1,3,7 >> gpurun_out/c17_ab.jsonl 2>>gpurun_out/c17_ab.err
$A --config c4 --libs base,_rs0 --flags 1 >> gpurun_out/c17_ab.jsonl 2>>gpurun_out/c17_ab.err
$A --config c5 --libs base,_rs0 --flags 1 >> gpurun_out/c17_ab.jsonl 2>>gpurun_out/c17_ab.err
echo done
