"""Summarise ncu reports / launch lists brought back in gpurun_out/ into profiles/.

    python scripts/ncu_summary.py TAG launches.csv prof1.ncu-rep [prof2.ncu-rep ...]

Writes profiles/TAG_launches.txt (per-kernel time and share of the captured
launches) and, per report, profiles/TAG_<name>.txt (key raw metrics) plus the
full raw page as CSV (profiles/TAG_<name>_raw.csv).
"""
import collections
import csv
import json
import io
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__average_warp_latency_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_membar",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_sample_count"]
UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path, out):
    txt = open(path).read().splitlines()
    i = [j for j, l in enumerate(txt) if l.startswith('"ID"')][0]
    agg = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO("\n".join(txt[i:]))):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", "")) * UNIT[r["Metric Unit"]]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none ({os.path.basename(path)})\n")
        fh.write("# cold-cache, serialised launches: compare SHARES, not absolutes\n")
        fh.write(f"{'kernel':64s} {'launches':>8s} {'total_us':>12s} {'share':>7s}\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{k:64s} {n:8d} {t:12.1f} {100 * t / tot:6.2f}%\n")
        fh.write(f"{'TOTAL':64s} {'':8s} {tot:12.1f}\n")


def report(path, out_txt, out_csv):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    open(out_csv, "w").write(raw)
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    with open(out_txt, "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on ({os.path.basename(path)})\n")
        for r in rows[2:]:
            fh.write(f"\n## {r[h.index('Kernel Name')]}\n")
            for k in KEYS:
                if k in h:
                    fh.write(f"{k:60s} {r[h.index(k)]:>16s} {units[h.index(k)]}\n")
            if "dram__bytes_read.sum" in h:
                def mb(k):
                    v = float(r[h.index(k)].replace(",", ""))
                    u = units[h.index(k)]
                    return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[u]
                fh.write(f"{'traffic (dram read + write)':60s} {mb('dram__bytes_read.sum') + mb('dram__bytes_write.sum'):16.3f} MB\n")


def traffic_json(path):
    """profiles/traffic.json: {kernel short name: dram read + write bytes per launch}."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    if os.path.exists("profiles/traffic.json"):
        out = json.load(open("profiles/traffic.json"))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").replace("rafem::", "")
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[h.index(k)].replace(",", "")) * scale[units[h.index(k)]]
        out[name] = tot
    json.dump(out, open("profiles/traffic.json", "w"), indent=1)


def main():
    tag = sys.argv[1]
    os.makedirs("profiles", exist_ok=True)
    for p in sys.argv[2:]:
        name = os.path.basename(p).rsplit(".", 1)[0]
        if p.endswith(".csv"):
            launches(p, f"profiles/{tag}_{name}.txt")
        else:
            report(p, f"profiles/{tag}_{name}.txt", f"profiles/{tag}_{name}_raw.csv")
            traffic_json(p)


if __name__ == "__main__":
    main()
