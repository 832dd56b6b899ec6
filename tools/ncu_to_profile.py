"""Turn one `ncu --set full` capture of k_check_scan into the committed
evidence: profiles/ncu_<config>[_<shadow>]_check_scan.json (read by bench.py
for roofline.traffic) and a details text file.
usage: python tools/ncu_to_profile.py <rep> <config> <fused 0/1> <details-out> [suffix] [kernel]
(kernel k_prop_waves -> profiles/ncu_<config>_<suffix>_prop_waves.json, read by bench.py --track)"""
import csv
import io
import json
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, config, fused, details_out, suffix="", kernel="k_check_scan"):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    d = dict(zip(raw[0], raw[2]))
    unit = dict(zip(raw[0], raw[1]))

    def val(k, scale_to=None):
        v = float(d[k].replace(",", ""))
        u = unit.get(k, "")
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
        return v * mult

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    out = {"kernel": kernel, "config": config, "fused": bool(int(fused)),
           "shadow": suffix or "bytes",
           "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
           "duration_ms_ncu": val("gpu__time_duration.sum"),
           "source": f"ncu --set full --clock-control none ({rep}); details in {details_out}",
           "registers": int(float(d["launch__registers_per_thread"])),
           "grid": int(float(d["launch__grid_size"])), "block": int(float(d["launch__block_size"])),
           "warp_instructions": float(d["smsp__inst_executed.sum"].replace(",", "")),
           "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
           "issue_active_pct": float(d["sm__inst_issued.avg.pct_of_peak_sustained_active"])}
    name = f"profiles/ncu_{config}{'_' + suffix if suffix else ''}_{kernel[2:]}.json"
    json.dump(out, open(name, "w"), indent=1)
    with open(details_out, "w") as f:
        f.write(ncu(rep, "--page", "details"))
    print(name, out["dram_bytes_per_launch"], out["duration_ms_ncu"])


if __name__ == "__main__":
    main(*sys.argv[1:])
