#!/bin/bash
# Round profile, part 1: full bench, reference arm, launch list.
# Part 2 (ncu --set full captures, one per gpurun call to stay under the
# 64 MiB gpurun_out limit): bash tools/ncu_full.sh tlog1p:64:pow10c_64
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --headline-only"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
tail -c 600 gpurun_out/bench_full.log; echo; cat gpurun_out/bench_ref.log
