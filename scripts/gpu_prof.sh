#!/bin/bash
# ncu evidence: launch list of one timed round + one --set full capture of the top kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SKIP=${SKIP:-2850}
COUNT=${COUNT:-960}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c $COUNT --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "launches exit $?"
if [ -n "$KREGEX" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -s ${KSKIP:-5} -c ${KCOUNT:-1} \
  -o gpurun_out/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
fi
ls -la gpurun_out
