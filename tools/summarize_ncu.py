"""Summarise ncu output for profiles/: a launch list (--metrics
gpu__time_duration.sum --csv --log-file) or a --set full report (.ncu-rep).

  python tools/summarize_ncu.py launches <csv> [title]   -> markdown table
  python tools/summarize_ncu.py full <ncu-rep> [title]   -> markdown table
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, title):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0].strip()].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"## {title}", "", f"source: `{path}` (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
           "| kernel | launches | total us | share | median us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        v = sorted(v)
        out.append(f"| `{k[:80]}` | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% | {v[len(v)//2]/1e3:.2f} |")
    return "\n".join(out)


WANT = [("gpu__time_duration.sum", "time"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
        ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("smsp__inst_executed.sum", "warp instr"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit %"), ("lts__t_sector_hit_rate.pct", "L2 hit %")]


def full(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lab = [f"{w[1]} ({units[hdr.index(w[0])]})" if w[0] in hdr and units[hdr.index(w[0])] else w[1] for w in WANT]
    out = [f"## {title}", "", f"source: `{path}` (ncu --set full)", "",
           "| kernel | " + " | ".join(lab) + " | top stalls |",
           "|---" * (len(WANT) + 2) + "|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        cells = []
        for key, _ in WANT:
            try:
                v = float(r[hdr.index(key)].replace(",", ""))
                cells.append(f"{v:.4g}")
            except (ValueError, IndexError):
                cells.append("-")
        stalls = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
                  float(r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                  and r[i] not in ("", "n/a")}
        top = ", ".join(f"{k} {v:.1f}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:3])
        out.append(f"| `{name[:60]}` | " + " | ".join(cells) + f" | {top} |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else path
    print(launches(path, title) if mode == "launches" else full(path, title))
