"""Summarise `ncu --set full` reports into the per-launch CSV bench.py and
profiles/ read: kernel, time_us, DRAM read / write bytes, DRAM %, tensor-pipe %,
SM %, registers, grid, block.

  python tools/ncu_summary.py out.csv rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

COLS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us (ncu reports usecond or nsecond: unit-checked below)
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "block": ("launch__block_size", 1.0),
}
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "%": 1.0, "": 1.0, "register/thread": 1.0, "block": 1.0, "thread": 1.0}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")}
        for k, (m, _) in COLS.items():
            v = d.get(m, "")
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                rec[k] = ""
                continue
            scale = SCALE.get(u.get(m, ""), 1.0)
            rec[k] = x * scale if k in ("time_us", "dram_read_bytes", "dram_write_bytes") else x
        yield rec


def main():
    out = sys.argv[1]
    recs = [r for rep in sys.argv[2:] for r in rows_of(rep)]
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["kernel"] + list(COLS))
        w.writeheader()
        w.writerows(recs)
    print(f"{len(recs)} launches -> {out}")


if __name__ == "__main__":
    main()
