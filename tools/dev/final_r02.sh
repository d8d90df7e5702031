#!/bin/bash
# round-2 end: the GPU test suite, then the measurement capture (tools/capture_r02.sh)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
bash tools/capture_r02.sh
