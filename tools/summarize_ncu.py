"""Summaries of ncu captures for profiles/ (run in the build container on gpurun_out/ files)."""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_thru_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_to_sm_sectors"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_base(v, unit):
    v = float(v.replace(",", ""))
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "hz": 1, "Khz": 1e3,
             "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1}
    return v * scale.get(unit, 1)


def full_report(rep, names):
    hdr, units, rows = raw_rows(rep)
    out = []
    for i, r in enumerate(rows):
        d = {"kernel": r[hdr.index("Kernel Name")][:60], "case": names[i] if i < len(names) else str(i)}
        for m, key in METRICS:
            if m in hdr:
                j = hdr.index(m)
                try:
                    d[key] = to_base(r[j], units[j])
                except ValueError:
                    d[key] = r[j]
        out.append(d)
    return out


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hdr = None
    data = collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data[d["ID"]]["kernel"] = d["Kernel Name"]
            data[d["ID"]][d["Metric Name"]] = to_base(d["Metric Value"], d["Metric Unit"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in data.values():
        name = d["kernel"].split("(")[0].replace("void ", "")[:48]
        a = agg[name]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    return agg


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "full":
        print(json.dumps(full_report(sys.argv[2], sys.argv[3].split(",")), indent=1))
    else:
        agg = launches(sys.argv[2])
        tot = sum(v[1] for v in agg.values())
        print(f"{'kernel':50s} {'n':>3s} {'total us':>9s} {'share':>6s} {'avg us':>8s} {'GB/s':>8s}")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            print(f"{k:50s} {v[0]:3d} {v[1]*1e6:9.1f} {100*v[1]/tot:5.1f}% {v[1]*1e6/v[0]:8.1f} {v[2]/v[1]/1e9 if v[1] else 0:8.0f}")
        print(f"{'total':50s}     {tot*1e6:9.1f}")
