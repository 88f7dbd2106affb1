"""Export ncu --set full captures (gpurun_out/prof_<tag>_<cfg>.ncu-rep) into profiles/:
<tag>_ncu_full_<cfg>_raw.csv, <tag>_ncu_full_<cfg>_details.csv, and the per-launch DRAM traffic
table profiles/ncu_traffic.json that bench.py reports as roofline.traffic.

usage: python tools/ncu_summarize.py <tag> [cfg ...]      (default cfgs: C2 C3 C4)
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALGO = {"C2": 2 * 10_000_000 * 80, "C3": 2 * 50_000_000 * 320, "C3R": 2 * 50_000_000 * 320, "C4": 2 * 59_652_323 * 36,
        "C5": 2 * 107_374_182 * 80, "C4M": 2 * 59_652_323 * 12, "P1": 2 * 16_777_216 * 36, "P2": 2 * 8_388_608 * 128}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0, "%": 1.0}


def export(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True,
                          check=True).stdout


def main():
    tag = sys.argv[1]
    def have(c):
        return any(os.path.exists(os.path.join(ROOT, "gpurun_out", f)) for f in
                   (f"prof_{tag}_{c}.ncu-rep", f"prof_{tag}_{c}_raw.csv"))
    cfgs = sys.argv[2:] or [c for c in ALGO if have(c)]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    for cfg in cfgs:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{cfg}.ncu-rep")
        if os.path.exists(rep):
            raw, details = export(rep, "raw"), export(rep, "details")
        else:   # exported on the GPU box (profile_round.sh), the report itself not brought back
            base = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_{cfg}")
            raw, details = open(base + "_raw.csv").read(), open(base + "_details.csv").read()
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{cfg}_raw.csv"), "w") as f:
            f.write(raw)
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{cfg}_details.csv"), "w") as f:
            f.write(details)
        rows = list(csv.reader(raw.splitlines()))
        hdr, units, vals = rows[0], rows[1], rows[2]

        def get(k):
            i = hdr.index(k)
            return float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)

        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        t = get("gpu__time_duration.sum")
        table[cfg] = {
            "kernel": vals[hdr.index("Kernel Name")],
            "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
            "gpu_time_s": t,
            "dram_pct_of_peak": get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers_per_thread": get("launch__registers_per_thread"),
            "algorithmic_bytes_per_launch": ALGO[cfg],
            "traffic_over_algorithmic": (rd + wr) / ALGO[cfg],
            "source": f"profiles/{tag}_ncu_full_{cfg}_raw.csv (ncu --set full --clock-control none, one launch)",
        }
        print(cfg, json.dumps(table[cfg]))
    # in-place C2 (profile_round.sh: ncu of tools/inplace_probe.py --cases C2, both directions):
    # dram bytes of all in-place kernels per step, averaged over the captured steps
    ip = os.path.join(ROOT, "gpurun_out", f"prof_{tag}_inplace_raw.csv")
    if os.path.exists(ip):
        raw = open(ip).read()
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_inplace_raw.csv"), "w") as f:
            f.write(raw)
        rows = list(csv.reader(raw.splitlines()))
        hdr, units = rows[0], rows[1]
        tot, t_s, steps = 0.0, 0.0, 0
        for vals in rows[2:]:
            def g(k):
                i = hdr.index(k)
                return float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            tot += g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
            t_s += g("gpu__time_duration.sum")
            steps += "ip_cycle_shift" in vals[hdr.index("Kernel Name")]
        if steps:
            table["C2_inplace"] = {"kernels": "ip_tile_kernel + ip_cycle_save_kernel + ip_cycle_shift_kernel",
                                   "dram_bytes_per_launch": tot / steps, "gpu_time_s_per_step": t_s / steps,
                                   "steps_captured": steps, "algorithmic_remap_bytes_per_step": ALGO["C2"],
                                   "source": f"profiles/{tag}_ncu_full_inplace_raw.csv (ncu --set full, C2 in place "
                                             "both directions)"}
            print("C2_inplace", json.dumps(table["C2_inplace"]))
    with open(path, "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()
