#!/bin/bash
# usage: bash tools/ncu_full.sh spec [spec...]   (spec = fn:width:dist); writes gpurun_out/full_<spec>.ncu-rep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python tools/ncu_target.py --n ${N:-16777216} "$@" > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for s in "$@"; do
  f=$(echo $s | tr : _)
  ncu --set full --import-source on --clock-control none -k regex:k_eval -s 2 -c 1 -o gpurun_out/full_$f python tools/ncu_target.py --n ${N:-16777216} $s > gpurun_out/ncu_full_$f.log 2>&1; echo "$f rc=$?"
done
