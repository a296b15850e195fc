#!/bin/bash
# GPU parity tests (stop at first failure) + per-kernel rates of the in-tree build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --tb=short -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
bash tools/variant_rates.sh paper_1502_05216_b200/lib/libtwofold_b200.so "$@"
