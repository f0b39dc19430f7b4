"""Summarise ncu outputs into profiles/ (run here, no GPU needed).
    python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep       > profiles/rNN_ncu_full.md
    python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep    # updates profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _csv(text):
    lines = [l for l in text.splitlines() if not l.startswith("==")]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path):
    rows = _csv(open(path).read())
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        k = r[ki]
        k = k[:k.index("(")] if "(" in k else k
        agg.setdefault(k, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total ms | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k[-90:]}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/1e6:.3f} | {sum(v)/tot*100:.1f}% |")


def _raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = _csv(out)
    return rows[0], rows[1], rows[2:]


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "launch__shared_mem_per_block_dynamic"]


def full(rep):
    h, units, rows = _raw(rep)
    ki = h.index("Kernel Name")
    print(f"ncu --set full capture `{os.path.basename(rep)}` (clock-control none)\n")
    for r in rows:
        print(f"### `{r[ki][:100]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"| {w} | {r[i]} | {units[i]} |")
        stalls = []
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1
        print("\nTop warp stall reasons (pc sampling): " +
              ", ".join(f"{n} {v/tot*100:.0f}%" for v, n in sorted(stalls, reverse=True)[:6]) + "\n")


def traffic(rep, key_upd="fused_update/llama2-7b/g2/w1", key_norm="probe/llama2-7b/w1"):
    h, units, rows = _raw(rep)
    ki = h.index("Kernel Name")
    def gb(r, m):
        i = h.index(m)
        v = float(r[i].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[units[i]]
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    for r in rows:
        t = gb(r, "dram__bytes_read.sum") + gb(r, "dram__bytes_write.sum")
        key = key_upd if ("ILb1E" in r[ki] or "_kernel<1" in r[ki]) else key_norm
        d[key] = t
    json.dump(d, open(p, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])
