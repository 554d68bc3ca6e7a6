"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py ROUND name=path.ncu-rep[:alg_bytes_or_flops] ... [--launches csv]

Writes profiles/ncu_<ROUND>_summary.md (human) and merges per-kernel numbers
into profiles/ncu_decode_summary.json (read by bench.py for `traffic`).
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "msecond": 1e-3, "second": 1.0}


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:120]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
                d[m + ".unit"] = units[i]
        res.append(d)
    return res


def main():
    rnd = sys.argv[1]
    specs = [a for a in sys.argv[2:] if "=" in a]
    launches = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    summary_path = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    md = [f"# ncu summary, round {rnd}", "",
          "One `ncu --set full --clock-control none --import-source on` capture per kernel "
          "(cold cache, serialised replay: shares and traffic are meaningful, absolute times are not "
          "bench numbers).", "",
          "| capture | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | algorithmic | DRAM % peak | "
          "SM % | tensor pipe % | regs | grid |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for spec in specs:
        name, rest = spec.split("=", 1)
        path, _, alg = rest.partition(":")
        for d in raw(path):
            t = d.get("gpu__time_duration.sum", 0.0)
            rd = d.get("dram__bytes_read.sum", 0.0)
            wr = d.get("dram__bytes_write.sum", 0.0)
            alg_s = ""
            entry = {"kernel": d["kernel"], "time_s": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "dram_bytes_per_launch": rd + wr,
                     "dram_pct_peak": d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     "sm_pct": d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "tensor_pct": d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                     "registers": d.get("launch__registers_per_thread"), "grid": d.get("launch__grid_size"),
                     "round": rnd}
            if alg:
                a = float(alg)
                entry["algorithmic"] = a
                # prefill (tensor-bound) captures carry FLOPs, decode ones bytes
                alg_s = f"{a / 1e9:.1f} GFLOP" if name.startswith("c4") else f"{a / 1e6:.1f} MB"
            summary[name] = entry
            md.append(f"| {name} | `{d['kernel'][:60]}` | {t * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                      f"{alg_s} | {entry['dram_pct_peak'] or 0:.1f} | {entry['sm_pct'] or 0:.1f} | "
                      f"{entry['tensor_pct'] or 0:.1f} | {entry['registers'] or 0:.0f} | {entry['grid'] or 0:.0f} |")
    if launches:
        rows = list(csv.reader(open(launches)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        agg = {}
        for r in rows[hdr + 1:]:
            if len(r) != len(h):
                continue
            k = r[h.index("Kernel Name")][:70]
            v = float(r[h.index("Metric Value")].replace(",", ""))
            agg.setdefault(k, []).append(v)
        tot = sum(sum(v) for v in agg.values())
        md += ["", f"Launch list (`{os.path.basename(launches)}`, gpu__time_duration, all launches of the run "
               "incl. setup):", "", "| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{rnd}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
