#!/bin/bash
# round 2 (session 4) first GPU call: per-class baseline on every config + staged-ring / CTA-H A/B
mkdir -p gpurun_out
A="timeout 1200 python tools/ab.py --class-work --reps 2"
$A --config c5 --libs base,_c1ring2,_c1ring2m2,_c1ring3,_hcta --flags 1 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
$A --config c4 --libs base,_c1ring2,_c1ring2m2,_c1ring3,_hcta --flags 1 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
$A --config c4 --ordering split --flags 1 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
$A --config c4 --algo app --flags 1 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
$A --config c3 --flags 0,1 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
$A --config c2 --flags 1,3,7 >> gpurun_out/c1_ab.jsonl 2>>gpurun_out/c1_ab.err
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c1_pytest.log
echo done
