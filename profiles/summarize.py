"""Summarise ncu outputs into the text files kept under profiles/ (run on the CPU box).

usage: python profiles/summarize.py launches <launches.csv> <out.txt>
       python profiles/summarize.py full <report.ncu-rep> <out.txt>
       python profiles/summarize.py traffic <report.ncu-rep> <workload> <family> <ncu_traffic.json> [index]
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)\n"
                f"# source: {path}; total {T / 1e6:.3f} ms over {sum(cnt.values())} launches\n")
        f.write(f"{'kernel':48s} {'launches':>8s} {'total_ms':>10s} {'share':>7s} {'avg_us':>9s}\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"{k:48s} {cnt[k]:8d} {v / 1e6:10.3f} {v / T:7.3f} {v / cnt[k] / 1e3:9.1f}\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, data = rows[0], rows[1], rows[2:]
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none; source {path}\n")
        for r in data:
            f.write(r[h.index("Kernel Name")][:100] + "\n")
            for w in WANT:
                if w in h:
                    i = h.index(w)
                    f.write(f"    {w:70s} {r[i]:>16s} {units[i]}\n")




def traffic(rep, workload, family, out_json, index="0"):
    """Record dram__bytes_read.sum + dram__bytes_write.sum of the first kernel in an ncu report
    as the per-launch traffic of a kernel family (read by bench.py's roofline.traffic)."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2 + int(index)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(v[i].replace(",", "")) * scale[units[i]]
    name = v[h.index("Kernel Name")].split("(")[0]
    t = json.load(open(out_json)) if os.path.exists(out_json) else {}
    t.setdefault(workload, {})[family] = {"dram_bytes": tot, "kernel": name,
                                          "source": f"{os.path.basename(rep)} launch {index}"}
    json.dump(t, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
