"""Copy the judged summaries of a profile round (tools/profile_round.sh) from
gpurun_out/ into profiles/ with the round prefix, and refresh
profiles/ncu_traffic.json from the ncu --set full captures."""
import json
import os
import subprocess
import sys

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r01"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24     # elements per captured launch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


# each part is optional: a capture-only call (tools/ncu_full.sh) has no bench logs
for bl in ("bench_full.log", "bench.log"):
    if os.path.exists(f"{G}/{bl}"):
        json.dump(last_json(f"{G}/{bl}"), open(f"{P}/{ROUND}_bench.json", "w"), indent=1)
        break
if os.path.exists(f"{G}/bench_ref.log"):
    json.dump(last_json(f"{G}/bench_ref.log"), open(f"{P}/{ROUND}_bench_reference.json", "w"), indent=1)
if os.path.exists(f"{G}/launches.csv"):
    lines = [ln for ln in open(f"{G}/launches.csv") if not ln.startswith("==")]
    open(f"{P}/{ROUND}_launches.csv", "w").writelines(lines)
TPATH = f"{P}/ncu_traffic.json"
traffic = json.load(open(TPATH)) if os.path.exists(TPATH) else {}   # merged per capture
for name in sorted(os.listdir(G)):
    if not (name.startswith("full_") and name.endswith(".ncu-rep")):
        continue
    tag = name[len("full_"):-len(".ncu-rep")]
    fn, width, dist = tag.split("_", 2)
    n = N
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                           os.path.join(G, name), str(n)], capture_output=True, text=True).stdout
    open(f"{P}/{ROUND}_ncu_full_{tag}.txt", "w").write(summ)
    det = subprocess.run(["ncu", "-i", os.path.join(G, name), "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    open(f"{P}/{ROUND}_ncu_details_{tag}.csv", "w").write(det)
    raw = subprocess.run(["ncu", "-i", os.path.join(G, name), "--page", "raw", "--csv",
                          "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout.splitlines()
    hdr = [h.strip('"') for h in raw[0].split('","')]
    unit = [u.strip('"') for u in raw[1].split('","')]
    val = [v.strip('"') for v in raw[2].split('","')]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(val[hdr.index("dram__bytes_read.sum")].replace(",", "")) * scale[unit[hdr.index("dram__bytes_read.sum")]]
    wr = float(val[hdr.index("dram__bytes_write.sum")].replace(",", "")) * scale[unit[hdr.index("dram__bytes_write.sum")]]
    ty = "double" if width == "64" else "float"
    key = f"cfg5_{fn}_f64" if dist in ("exp64s", "logu64s") else f"k_eval<{ty},{fn}>"
    traffic[key] = {
        "dram_read_bytes": rd, "dram_write_bytes": wr, "elements": n,
        "algorithmic_bytes": n * (32 if width == "64" else 16),
        "source": f"profiles/{ROUND}_ncu_full_{tag}.txt (ncu --set full)",
        "traffic_bytes": rd + wr}
json.dump(traffic, open(TPATH, "w"), indent=1)
print("saved", sorted(traffic))
