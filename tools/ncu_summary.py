"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches FILE.csv      # per-kernel launch list stats
  python tools/ncu_summary.py full FILE.ncu-rep      # key metrics per captured kernel
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "tmem_pipe_%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    d = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rec = dict(zip(hdr, r))
            if rec.get("Metric Name") == "gpu__time_duration.sum":
                name = rec["Kernel Name"].split("(")[0].split("::")[-1]
                unit = rec.get("Metric Unit", "ns")
                v = float(rec["Metric Value"].replace(",", ""))
                d[name].append(v * (1e-3 if unit in ("ns", "nsecond") else 1.0))
    tot = sum(sum(v) for v in d.values())
    print(f"{'kernel':36s} {'launches':>8s} {'mean us':>10s} {'share':>7s}")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:36s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v) / tot:7.1%}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        name = rec["Kernel Name"].split("(")[0].split("::")[-1]
        print(f"== {name} ({rec.get('Kernel Name', '')[:90]})")
        for key, short in KEYS:
            if key in rec:
                u = units[hdr.index(key)]
                print(f"   {short:14s} {rec[key]:>16s} {u}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
