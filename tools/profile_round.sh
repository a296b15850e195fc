#!/bin/bash
# Round profile: full bench, reference arm, launch list, ncu --set full of the headline kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --headline-only"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
for s in tlog1p:64:pow10c_64 texpm1:64:pow10_64 tlog1p:32:log32; do
  f=$(echo $s | tr : _)
  python tools/ncu_target.py $s > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:k_eval -s 2 -c 1 -o gpurun_out/full_$f python tools/ncu_target.py $s > gpurun_out/ncu_full_$f.log 2>&1; echo "full $f rc=$?"
done
tail -c 600 gpurun_out/bench_full.log; echo; cat gpurun_out/bench_ref.log
