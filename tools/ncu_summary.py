"""Summarise an `ncu --set full` report (one line block per profiled launch).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json --pick N]

Prints the metrics the roofline discussion in DESIGN.md uses: duration, DRAM
bytes, achieved DRAM bandwidth, DMMA (FP64 tensor) pipe activity, occupancy,
shared-memory bank conflicts and the top warp stall reasons.  With --json, the
launch `--pick` (default: the longest) is written as the `traffic` source that
bench.py reads (dram_bytes_per_launch).
"""
import argparse
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("Grid Size", "grid"),
    ("Block Size", "block"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
     "dmma_active_pct(active SMs)"),
    ("sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "fp64_tensor_pct_elapsed"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
         "usecond": 1e-6, "us": 1e-6, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def value(hdr, units, row, key):
    if key not in hdr:
        return None, ""
    i = hdr.index(key)
    v = row[i].replace(",", "")
    try:
        return float(v), units[i]
    except ValueError:
        return row[i], units[i]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--pick", type=int, default=-1)
    a = ap.parse_args()
    hdr, units, data = load(a.rep)
    stall_cols = [i for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled_")
                  or h.startswith("smsp__pcsamp_warps_issue_stalled_")]
    durations = []
    for n, row in enumerate(data):
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"--- launch {n}: {name[:110]}")
        rec = {}
        for key, label in KEYS:
            v, u = value(hdr, units, row, key)
            if v is None:
                continue
            rec[label] = (v, u)
            print(f"  {label:32s} {v} {u}")
        d, du = rec.get("duration", (0.0, "us"))
        rd, ru = rec.get("dram_read", (0.0, "byte"))
        wr, wu = rec.get("dram_write", (0.0, "byte"))
        secs = float(d) * SCALE.get(du, 1e-6)
        byts = float(rd) * SCALE.get(ru, 1) + float(wr) * SCALE.get(wu, 1)
        if secs > 0:
            print(f"  {'dram_GBps':32s} {byts / secs / 1e9:.1f}")
        durations.append((secs, byts, name))
        stalls = []
        for i in stall_cols:
            try:
                stalls.append((float(row[i].replace(",", "")), hdr[i]))
            except ValueError:
                pass
        stalls.sort(reverse=True)
        for v, h in stalls[:5]:
            print(f"  stall {h.split('stalled_')[-1]:26s} {v:.3f}")
    if a.json and durations:
        k = a.pick if a.pick >= 0 else max(range(len(durations)), key=lambda i: durations[i][0])
        secs, byts, name = durations[k]
        json.dump({"kernel": name, "duration_s": secs, "dram_bytes_per_launch": byts,
                   "source": a.rep}, open(a.json, "w"), indent=1)
        print("wrote", a.json, "launch", k)


if __name__ == "__main__":
    sys.exit(main())
