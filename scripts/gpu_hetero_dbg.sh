#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python scripts/hetero_emulation.py --clients 1000 --out gpurun_out/h_new.json > gpurun_out/h_new.log 2>&1; echo "new rc=$?"; tail -1 gpurun_out/h_new.log
if [ -d _old ]; then
  (cd _old && python -c "import __graft_entry__ as g; g.build()" > ../gpurun_out/h_oldbuild.log 2>&1 && timeout 600 python scripts/hetero_emulation.py --clients 1000 --out ../gpurun_out/h_old.json > ../gpurun_out/h_old.log 2>&1; echo "old rc=$?"; tail -1 ../gpurun_out/h_old.log)
fi
