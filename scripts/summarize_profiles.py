"""Local step after scripts/refresh_profiles.sh ran on the GPU box: copy the
bench lines and summarise the ncu captures of gpurun_out/prof/ into
profiles/ (r01_bench_c*.json, r01_launches_c1*, r01_ncu_full_*.txt,
ncu_traffic.json).  python scripts/summarize_profiles.py [round-tag]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def last_json(path):
    for line in reversed(open(path).read().strip().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    raise ValueError(path)


for src, dst in [("bench_c1", "bench_c1"), ("bench_c2", "bench_c2"), ("bench_c3", "bench_c3"),
                 ("bench_c4", "bench_c4"), ("bench_ref_c1", "bench_reference_c1")]:
    f = os.path.join(SRC, src + ".json")
    if os.path.exists(f):
        json.dump(last_json(f), open(os.path.join(DST, f"{tag}_{dst}.json"), "w"), indent=1)

lc = os.path.join(SRC, "launches_c1.csv")
if os.path.exists(lc):
    subprocess.run(["cp", lc, os.path.join(DST, f"{tag}_launches_c1.csv")], check=True)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_summary.py"), lc],
                         capture_output=True, text=True).stdout
    open(os.path.join(DST, f"{tag}_launches_c1_summary.json"), "w").write(out)


def summary(rep):
    js = rep + ".json"
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "--json", js],
                         capture_output=True, text=True).stdout
    return txt, json.load(open(js))


def dram(d):
    def val(s):
        num, unit = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        return float(num) * scale
    tdur = d.get("gpu__time_duration.sum", "0 ns").split()
    us = float(tdur[0]) * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(tdur[1], 1)
    return val(d["dram__bytes_read.sum"]) + val(d["dram__bytes_write.sum"]), us


traffic = {"_note": "DRAM bytes (read + write) per launch of the dominant kernels, one ncu --set full "
                    "capture of one launch each (scripts/refresh_profiles.sh, scripts/summarize_profiles.py); "
                    "keyed by bench config, then phase (config4 'batched': mean of its two kernels, the "
                    "phase launches both).  Durations under ncu are cold-cache and serialised."}
c1 = {"chol_factor_kernel": "chol_factor", "chol_backsolve_kernel": "chol_solve", "lsqr_cluster_kernel": "lsqr",
      "gram_exact_kernel": "gram", "dual_kernel": "dual", "decide_kernel": "decide"}
txt1, txt4 = [], []
for k, ph in c1.items():
    rep = os.path.join(SRC, f"full_c1_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    t, d = summary(rep)
    txt1.append(t)
    for _, v in d.items():
        b, us = dram(v)
        traffic.setdefault("config1", {})[ph] = {"dram_bytes_per_launch": b, "duration_us_under_ncu": round(us, 2)}
if txt1:
    open(os.path.join(DST, f"{tag}_ncu_full_c1.txt"), "w").write(
        "=== config 1: dominant kernels (ncu --set full, one launch each)\n" + "".join(txt1))
rep = os.path.join(SRC, "full_c2_chol_factor_kernel.ncu-rep")
if os.path.exists(rep):
    t, d = summary(rep)
    open(os.path.join(DST, f"{tag}_ncu_full_c2_chol_factor.txt"), "w").write(
        "=== config 2: chol_factor_kernel (ncu --set full, one launch)\n" + t)
    for _, v in d.items():
        b, us = dram(v)
        traffic.setdefault("config2", {})["chol_factor"] = {"dram_bytes_per_launch": b,
                                                            "duration_us_under_ncu": round(us, 2)}
bsum, usum, nk = 0.0, 0.0, 0
for k in ("batched_kernel", "batched_lsqr_kernel"):
    rep = os.path.join(SRC, f"full_c4_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    t, d = summary(rep)
    txt4.append(t)
    for _, v in d.items():
        b, us = dram(v)
        bsum, usum, nk = bsum + b, usum + us, nk + 1
if nk:
    traffic["config4"] = {"batched": {"dram_bytes_per_launch": bsum / nk, "duration_us_under_ncu": round(usum / nk, 2)}}
    open(os.path.join(DST, f"{tag}_ncu_full_c4.txt"), "w").write(
        "=== config 4: batched_kernel + batched_lsqr_kernel (ncu --set full, one launch each)\n" + "".join(txt4))
json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
print("profiles updated:", sorted(os.listdir(DST)))
