#!/bin/bash
# The driver's round-end GPU check, as one process: python -m pytest tests/ -x -q -m gpu (+ smoke)
mkdir -p gpurun_out
( time timeout 1500 python -m pytest tests/ -x -q -m gpu --durations=12 ) > gpurun_out/suite_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/suite_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/suite_smoke.log 2>&1
echo done
