#!/bin/bash
# kernel rates of alternative builds: bash tools/variant_rates.sh lib1.so lib2.so ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in $(seq ${REPS:-1}); do
for so in "$@"; do
  echo "== $so"
  TWOFOLD_B200_LIB=$so python bench.py --steps 20 --no-e2e --no-cpu --no-siblings --no-eft > gpurun_out/var.log 2>&1
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/var.log").read().strip().splitlines()[-1])
print("headline", round(d["value"] / 1e9, 2), {k: round(v["elements_per_s"] / 1e9, 1) for k, v in d["per_function"].items()})
PY
done
done
