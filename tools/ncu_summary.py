"""Per-kernel key metrics of an ncu --set full report -> JSON (profiles/).

    python tools/ncu_summary.py gpurun_out/prof_all_r10.ncu-rep profiles/r10_ncu_all_kernels.json
"""
import csv
import io
import json
import subprocess
import sys

M = {
    "gpu__time_duration.sum": ("us", 1.0),
    "sm__cycles_elapsed.max": ("kcyc", 1e-3),
    "sm__cycles_elapsed.avg.per_second": ("sm_ghz", 1.0),
    "dram__bytes_read.sum": ("dram_read_bytes", None),
    "dram__bytes_write.sum": ("dram_write_bytes", None),
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": ("tc_pipe_active_pct", 1.0),
    "lts__t_sector_hit_rate.pct": ("l2_hit_pct", 1.0),
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": ("dram_pct_of_peak", 1.0),
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": ("sm_pct_of_peak", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:60]}
        for k, (name, scale) in M.items():
            if k not in hdr:
                continue
            i = hdr.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if scale is None:
                v *= UNIT.get(units[i], 1)
            else:
                v *= scale
            d[name] = round(v, 3)
        if "dram_read_bytes" in d and "us" in d:
            d["dram_GBps"] = round((d["dram_read_bytes"] + d.get("dram_write_bytes", 0)) / (d["us"] * 1e-6) / 1e9, 1)
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(d)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
