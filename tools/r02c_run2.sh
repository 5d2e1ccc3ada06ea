#!/bin/bash
# short-row windows (W), x-chunk prefetch, producer-warp CTA kernels: A/B; parity of the new base; core decomposition test
mkdir -p gpurun_out
A="timeout 1200 python tools/ab.py --class-work --reps 2"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "core or golden or edge or giant" > gpurun_out/c2_pytest_core.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_pytest_core.log
$A --config c3 --libs base,_w2,_w8 --flags 0,1 >> gpurun_out/c2_ab.jsonl 2>>gpurun_out/c2_ab.err
$A --config c4 --libs base,_w2,_w8,_nopf,_pf,_pf2 --flags 1 >> gpurun_out/c2_ab.jsonl 2>>gpurun_out/c2_ab.err
$A --config c5 --libs base,_nopf,_pf,_pf2 --flags 1 >> gpurun_out/c2_ab.jsonl 2>>gpurun_out/c2_ab.err
$A --config c4 --algo app --libs base,_nopf --flags 1 >> gpurun_out/c2_ab.jsonl 2>>gpurun_out/c2_ab.err
$A --config c2 --libs base,_w2,_nopf,_pf --flags 1,3 >> gpurun_out/c2_ab.jsonl 2>>gpurun_out/c2_ab.err
echo done
