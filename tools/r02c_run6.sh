#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/dbg_lib.py _ra1 22 > gpurun_out/c7_dbg22.log 2>&1
timeout 300 python tools/dbg_lib.py _ra1 24 > gpurun_out/c7_dbg24.log 2>&1
echo done
