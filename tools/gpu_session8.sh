#!/bin/bash
# full-size parity (BASELINE configs, bench launch configuration) + smoke
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m "slow" -x > gpurun_out/pytest_slow.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_slow.log
echo done
