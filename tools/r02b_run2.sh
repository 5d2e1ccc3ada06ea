#!/bin/bash
# A/B of the staged-ring / CTA-H / hash-R variants on C5, C4, C3 (count + checksum)
mkdir -p gpurun_out
A="timeout 1200 python tools/ab.py --class-work --reps 2"
$A --config c5 --libs base,_c1ring2,_c1ring2m2,_hcta,_rhash --flags 1 >> gpurun_out/r2_ab.jsonl 2>>gpurun_out/r2_ab.err
$A --config c4 --libs base,_c1ring2,_c1ring2m2,_hcta,_rhash --flags 1 >> gpurun_out/r2_ab.jsonl 2>>gpurun_out/r2_ab.err
$A --config c3 --libs base,_rhash --flags 1 >> gpurun_out/r2_ab.jsonl 2>>gpurun_out/r2_ab.err
timeout 1500 python tools/c5_parity.py > gpurun_out/r2_c5_parity.json 2> gpurun_out/r2_c5_parity.err
echo done
