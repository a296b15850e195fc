#!/bin/bash
# kernel rates of alternative builds, alternating on one box:
#   bash tools/variant_rates.sh lib1.so lib2.so ...   (REPS=n rounds)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in $(seq ${REPS:-1}); do
for so in "$@"; do
  echo "== $so"
  TWOFOLD_B200_LIB=$so ROUNDS=1 python tools/rate_probe.py
done
done
