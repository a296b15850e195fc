#!/bin/bash
# quick GPU check: parity tests (stop at first failure) + kernel rates
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests -m gpu -q --tb=short -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 20 --no-e2e --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print("headline Gelem/s", round(d["value"] / 1e9, 2), {k: round(v, 4) for k, v in d["kernel_ms"].items()}, "frac", round(d["roofline"]["frac"], 3), d["clocks"])
for k, v in d["per_function"].items():
    print(f'{k:12s} {v["elements_per_s"]/1e9:7.1f} Gelem/s  fp_frac {v["fp_pipe_frac"]:.3f}  hbm_frac {v["hbm_frac"]:.3f}')
PY
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
for k, v in d.get("siblings", {}).items():
    r = [x for x in v if x.startswith("vs_")][0]
    print(f'{k:12s} {v["elements_per_s"]/1e9:7.1f} Gelem/s  {r} {v[r]:.3f}')
PY
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
for k, v in d.get("eft_ops", {}).items():
    print(f'{k:18s} {v["elements_per_s"]/1e9:7.1f} Gelem/s  {v["hbm_gbs"]:7.0f} GB/s  hbm_frac {v["hbm_frac"]:.3f}')
PY
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print("cfg1_small", d.get("cfg1_small"))
PY
