#!/bin/bash
# Full GPU test suite (+ smoke) on the current tree.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/u_smoke.log
timeout 2400 python -m pytest tests -q -m gpu -s ${PYARGS:-} > gpurun_out/u_gpu.log 2>&1; echo "gpu suite rc=$?"
grep -E "passed|failed|FAILED|C3:|C2:" gpurun_out/u_gpu.log | tail -12
