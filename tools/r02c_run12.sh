#!/bin/bash
# class G: giant rows streamed by the whole CTA - parity and timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "giant or golden or hub or scaled or wide or shrunk" > gpurun_out/c14_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c14_pytest.log
A="timeout 900 python tools/ab.py --class-work --reps 3"
$A --config c4 --ordering split --flags 1 >> gpurun_out/c14_ab.jsonl 2>>gpurun_out/c14_ab.err
$A --config c4 --algo app --flags 1 >> gpurun_out/c14_ab.jsonl 2>>gpurun_out/c14_ab.err
$A --config c4 --ordering split --algo app --flags 1 >> gpurun_out/c14_ab.jsonl 2>>gpurun_out/c14_ab.err
$A --config c2 --ordering split --flags 1 >> gpurun_out/c14_ab.jsonl 2>>gpurun_out/c14_ab.err
$A --config c4 --flags 1 >> gpurun_out/c14_ab.jsonl 2>>gpurun_out/c14_ab.err
echo done
