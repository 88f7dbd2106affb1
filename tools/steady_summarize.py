"""Add the steady-state DRAM traffic of back-to-back bench launches to profiles/ncu_traffic.json:
reads <tag>_steady_<cfg>.csv (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --cache-control none, launches in the middle of the bench's timed loop),
copies it to profiles/ and records read/write/ns per launch and their ratio to the algorithmic bytes.
Run after tools/ncu_summarize.py (which rewrites the one-launch entries).
usage: python tools/steady_summarize.py <tag> [cfg ...]"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summarize import ALGO  # noqa: E402


def main():
    tag = sys.argv[1]
    cfgs = sys.argv[2:] or list(ALGO)
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    table = json.load(open(path))
    for cfg in cfgs:
        src = os.path.join(ROOT, "gpurun_out", f"{tag}_steady_{cfg}.csv")
        if not os.path.exists(src):
            continue
        shutil.copy(src, os.path.join(ROOT, "profiles", f"{tag}_steady_{cfg}.csv"))
        rows = [r for r in csv.reader(open(src)) if len(r) == 15 and r[0] != "ID"]
        launches = {}
        for r in rows:
            launches.setdefault(r[0], {})[r[12]] = float(r[14].replace(",", ""))
        ls = [{"read": v["dram__bytes_read.sum"], "write": v["dram__bytes_write.sum"], "ns": v["gpu__time_duration.sum"]}
              for _, v in sorted(launches.items(), key=lambda kv: int(kv[0]))]
        if not ls:
            continue
        ratio = sum(x["read"] + x["write"] for x in ls) / len(ls) / ALGO[cfg]
        e = table.setdefault(cfg, {})
        e["steady_state_ratio"] = ratio
        e["steady_state_launches"] = ls
        e["steady_state_gbs"] = ALGO[cfg] / (sum(x["ns"] for x in ls) / len(ls)) 
        e["steady_state_source"] = (f"profiles/{tag}_steady_{cfg}.csv: ncu --metrics dram__bytes_read.sum,"
                                    "dram__bytes_write.sum,gpu__time_duration.sum --cache-control none "
                                    "--clock-control none, launches 5-7 of back-to-back bench steps")
        print(cfg, f"steady ratio {ratio:.4f}, {e['steady_state_gbs']:.0f} GB/s per launch")
    with open(path, "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()
