"""Turn the gpurun_out/ evidence of tools/profile_round.sh into the tracked
profiles/ summaries: bench lines, ncu launch-list shares, DAS ncu details and
its DRAM traffic (read by bench.py's roofline.traffic)."""
import collections
import csv
import json
import os
import shutil
import subprocess

OUT, PROF = "gpurun_out", "profiles"
WORKLOAD = "cfg2 PWI 128el x 11 angles x 2048 samples -> 512x512, DAS+envelope+dB30, linear"

shutil.copy(os.path.join(OUT, "bench_default.log"), os.path.join(PROF, "r01_bench_latest.jsonl"))
shutil.copy(os.path.join(OUT, "bench_reference.log"), os.path.join(PROF, "r01_bench_reference.jsonl"))

rows = [r for r in csv.reader(open(os.path.join(OUT, "launches.csv"))) if len(r) > 5]
hdr, data = rows[0], rows[1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    name = r[ik].split("(")[0]
    tot[name] += float(r[iv].replace(",", "")) * scale[r[iu]]
    cnt[name] += 1
s = sum(tot.values())
kern = [{"name": k, "launches": cnt[k], "total_us": round(v, 1),
         "us_per_launch": round(v / cnt[k], 1), "share_pct": round(v / s * 100, 2)}
        for k, v in sorted(tot.items(), key=lambda x: -x[1])]
json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none --csv "
                      "python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e",
           "note": "cold-cache, serialised per-launch times under ncu; compare SHARES with "
                   "bench.py, not absolute times", "kernels": kern},
          open(os.path.join(PROF, "r01_launches_tma.json"), "w"), indent=1)
for k in kern:
    print(f"{k['share_pct']:6.2f} %  {k['us_per_launch']:9.1f} us  {k['name'][:70]}")

rep = os.path.join(OUT, "prof_das_tma.ncu-rep")
txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
open(os.path.join(PROF, "r01_das_tma_ncu.txt"), "w").write(txt)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
r = list(csv.reader(raw))
d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rb = float(d["dram__bytes_read.sum"]) * mult[u["dram__bytes_read.sum"]]
wb = float(d["dram__bytes_write.sum"]) * mult[u["dram__bytes_write.sum"]]
name = [l for l in txt.splitlines() if "das_tma_kernel" in l][0].strip().split("(")[0]
json.dump({"workload": WORKLOAD, "interp": "linear", "kernel": name,
           "source": "profiles/r01_das_tma_ncu.txt (ncu --set full, 32 frames per launch)",
           "dram_bytes_read_per_launch": rb, "dram_bytes_write_per_launch": wb,
           "frames_per_launch": 32, "dram_bytes_per_frame": (rb + wb) / 32},
          open(os.path.join(PROF, "das_traffic.json"), "w"), indent=1)
for k in ("gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
          "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum"):
    print(k, d.get(k), u.get(k))
print("DRAM read/write MB", rb / 1e6, wb / 1e6, "kernel", name)
