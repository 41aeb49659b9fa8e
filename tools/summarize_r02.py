"""Round-2 evidence: turn gpurun_out/ (tools/profile_round.sh, ncu reports
already summarised on the box) into tracked profiles/r02_* files, and refresh
profiles/das_traffic.json (read by bench.py's roofline.traffic)."""
import collections
import csv
import gzip
import json
import os
import shutil

OUT, PROF = "gpurun_out", "profiles"
WORKLOAD = "cfg2 PWI 128el x 11 angles x 2048 samples -> 512x512, DAS+envelope+dB30, linear"
KEYS = ("gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum")
MULT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def copy(src, dst):
    if os.path.exists(os.path.join(OUT, src)):
        shutil.copy(os.path.join(OUT, src), os.path.join(PROF, dst))


def raw_metrics(stem):
    r = [row for row in csv.reader(open(os.path.join(OUT, stem + "_raw.csv"))) if row]
    d, u = dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))
    out = {k: f"{d[k]} {u.get(k, '')}".strip() for k in KEYS if k in d}
    stalls = {k.split("stalled_")[1]: int(float(v)) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k
              and v not in ("", "0")}
    out["stall_samples"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    out["kernel"] = d.get("Kernel Name", "")
    return out, d, u


def summarise(stem, dst):
    copy(stem + "_details.txt", dst + "_ncu.txt")
    m, _, _ = raw_metrics(stem)
    json.dump(m, open(os.path.join(PROF, dst + "_ncu.json"), "w"), indent=1)
    return m


copy("bench_default.log", "r02_bench_default.jsonl")
copy("bench_reference.log", "r02_bench_reference.jsonl")
copy("pt_gpu.log", "r02_pytest_gpu.log")
copy("smoke.log", "r02_smoke.log")
# the one-frame numbers come from the plain das1_probe run's log (its json is
# overwritten by the later run under ncu, whose timings are not bench values)
if os.path.exists(os.path.join(OUT, "das1.log")):
    one_frame = {}
    for line in open(os.path.join(OUT, "das1.log")):
        name, _, rest = line.strip().partition(" ")
        if rest.startswith("{"):
            one_frame[name] = json.loads(rest)
        elif name == "dropin":
            one_frame["dropin_fps_cfg2"] = float(rest)
    json.dump(one_frame, open(os.path.join(PROF, "r02_das_one_frame.json"), "w"), indent=1)
copy("k2_probe.json", "r02_k2_probe.json")

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
                      "python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stai",
           "note": "whole process (setup, warm-up and the timed steps), cold-cache and "
                   "serialised under ncu: compare SHARES with bench.py, not absolute times",
           "kernels": kern}, open(os.path.join(PROF, "r02_launches.json"), "w"), indent=1)
for k in kern:
    print(f"{k['share_pct']:6.2f} %  {k['us_per_launch']:9.1f} us  x{k['launches']}  {k['name'][:60]}")

das = summarise("prof_das_tma", "r02_das_tma")
_, d, u = raw_metrics("prof_das_tma")
rb = float(d["dram__bytes_read.sum"]) * MULT[u["dram__bytes_read.sum"]]
wb = float(d["dram__bytes_write.sum"]) * MULT[u["dram__bytes_write.sum"]]
json.dump({"workload": WORKLOAD, "interp": "linear", "kernel": das["kernel"],
           "source": "profiles/r02_das_tma_ncu.txt (ncu --set full, 32 frames per launch)",
           "dram_bytes_read_per_launch": rb, "dram_bytes_write_per_launch": wb,
           "frames_per_launch": 32, "dram_bytes_per_frame": (rb + wb) / 32},
          open(os.path.join(PROF, "das_traffic.json"), "w"), indent=1)
k2 = summarise("prof_k2", "r02_k2_fused")
one = summarise("prof_das1", "r02_das_one_frame")
for name, m in (("DAS 32 frames", das), ("K2+K3 fused", k2), ("DAS one frame", one)):
    print(name, m["kernel"][:70])
    for k in KEYS:
        if k in m:
            print("   ", k, m[k])
    print("    stalls", list(m["stall_samples"].items())[:6])
