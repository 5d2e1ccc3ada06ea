#!/bin/bash
# round-2 check 3: checksum gather variants and L2 evict_last for the hot rows
mkdir -p gpurun_out
timeout 900 python tools/ab.py --config c4 --libs _cks0,_cks1,_l2,_l2h32,_l2h96,_l2cks1 --flags 0,1 >> gpurun_out/ab3.jsonl 2>>gpurun_out/ab3.err
timeout 1200 python tools/ab.py --config c5 --libs _cks0,_cks1,_l2,_l2h96,_l2cks1 --flags 1 --reps 3 >> gpurun_out/ab3.jsonl 2>>gpurun_out/ab3.err
