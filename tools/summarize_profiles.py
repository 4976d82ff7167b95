"""Summarise a tools/round_profile.sh capture into profiles/.

    python tools/summarize_profiles.py gpurun_out/r1s3 r1s3

Writes profiles/<tag>_launch_shares.json (per-kernel launches, mean time and
share of our kernels' time from the ncu launch lists — cold-cache and
serialised, so shares, not bench values), profiles/<tag>_ncu_full_summary.json
(DRAM bytes, throughput and pipe utilisation per captured launch, from
`ncu -i <rep> --page raw --csv`) and copies the bench lines.
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__shared_mem_per_block_dynamic",
]


def launch_shares(path):
    rows = []
    with open(path) as fp:
        lines = [l for l in fp if not l.startswith("==")]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v / 1e3 if unit == "nsecond" else v
        rows.append((r["Kernel Name"], us))
    agg = collections.defaultdict(list)
    for name, us in rows:
        agg[name[:96]].append(us)
    total = sum(sum(v) for v in agg.values()) or 1.0
    return sorted(({"kernel": k, "launches": len(v), "mean_us": round(sum(v) / len(v), 2),
                    "share": round(sum(v) / total, 4)} for k, v in agg.items()),
                  key=lambda d: -d["share"])


def full_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rd = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rd[0], rd[1], rd[2:]
    res = []
    for row in data:
        d = {"Kernel Name": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{row[i]} {units[i]}".strip()
        res.append(d)
    return res


def _gbytes(v):
    num, unit = v.split()
    return float(num) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def update_traffic(full, tag):
    """profiles/decode_traffic.json: DRAM bytes per launch of each bench
    line's dominant kernel (read + write, from the full captures); bench.py
    puts them in the lines' roofline.traffic."""
    path = os.path.join(ROOT, "profiles", "decode_traffic.json")
    tj = json.load(open(path)) if os.path.exists(path) else {}
    picks = {"stack": ("stack_full", "decode_stack"), "layer_stack": ("layer_full", "decode_stack"),
             "prefill": ("prefill_full", "prefill_grouped")}
    for key, (cap, kname) in picks.items():
        for k in full.get(cap, []):
            if kname in k["Kernel Name"]:
                rd, wr = _gbytes(k["dram__bytes_read.sum"]), _gbytes(k["dram__bytes_write.sum"])
                pre = f"{key}_"
                tj[pre + "kernel"] = k["Kernel Name"]
                tj[pre + "dram_bytes_per_launch"] = int(rd + wr)
                tj[pre + "dram_bytes_read"] = int(rd)
                tj[pre + "dram_bytes_write"] = int(wr)
                tj[pre + "source"] = f"ncu --set full --clock-control none (profiles/{tag}_ncu_full_summary.json, {cap})"
                break
    json.dump(tj, open(path, "w"), indent=1)


def main():
    src, tag = sys.argv[1], sys.argv[2]
    prof = os.path.join(ROOT, "profiles")
    shares = {"note": "ncu --metrics gpu__time_duration.sum --clock-control none, our kernels only "
                      "(cold-cache, serialised): shares, not bench values"}
    for name in ("stack32", "prefill512"):
        p = os.path.join(src, f"launches_{name}.csv")
        if os.path.exists(p):
            shares[name] = launch_shares(p)
            shutil.copy(p, os.path.join(prof, f"{tag}_launches_{name}.csv"))
    json.dump(shares, open(os.path.join(prof, f"{tag}_launch_shares.json"), "w"), indent=1)
    full = {"note": "ncu --set full --clock-control none (cache flushed between replays): DRAM bytes "
                    "and pipe utilisation per launch; durations are cold-cache"}
    for name in ("stack_full", "layer_full", "prefill_full"):
        rep = os.path.join(src, f"{name}.ncu-rep")
        if os.path.exists(rep):
            full[name] = full_summary(rep)
    json.dump(full, open(os.path.join(prof, f"{tag}_ncu_full_summary.json"), "w"), indent=1)
    update_traffic(full, tag)
    for f in ("bench_stack32", "bench_prefill512", "bench_layer"):
        p = os.path.join(src, f + ".json")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(prof, f"{tag}_{f}.json"))
    print(json.dumps(shares, indent=1)[:3000])


if __name__ == "__main__":
    main()
