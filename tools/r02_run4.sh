#!/bin/bash
# round-2 check 4: per-class baselines of the secondary configs (base build)
mkdir -p gpurun_out
timeout 600 python tools/ab.py --config c4 --ordering split --algo apm --flags 0,1 --reps 2 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
timeout 600 python tools/ab.py --config c4 --ordering degree --algo app --flags 0,1 --reps 2 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
timeout 600 python tools/ab.py --config c2 --flags 0,1,3,7 --reps 3 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
timeout 600 python tools/ab.py --config c3 --flags 0,1 --reps 3 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
timeout 600 python tools/ab.py --config c2 --ordering split --algo app --flags 1 --reps 2 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
