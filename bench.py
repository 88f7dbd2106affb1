#!/usr/bin/env python
"""bench.py -- ADHA layout remap on B200: remap GB/s (read+write), bit-exact path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl adha|reference]

One step = one pass of the hot path over the configuration's records (SURVEY.md
8(d)).  The default is C5, the configuration BASELINE.json's metric is quoted on
("at 1/2/4/8 B200"): one AoS->SoA remap of 8 GiB of 80-byte records, split over
the GPUs.  Multi-GPU: one process per GPU (torchrun; `--gpus N` without torchrun
re-launches itself through torch.distributed.run with N ranks); the record array
is sharded by contiguous index range (adha_shard_range) with no collective on the
data path; each rank remaps its own shard ("strong" for C5: 8 GiB in total;
"weak" for the other configs, e.g. C2: 10M records per rank).
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0
GRAPH_STEPS = 16               # steps per CUDA-graph launch for launch-bound (< 256 MB) steps      # /opt/skills/guides/B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json

CONFIGS = {
    # name: (description, widths, src labels, dst labels chain, n_records, scaling)
    "C1": ("3-field float record (x,y,z), 1024 records, AoS->SoA->AoS", "xyz", 1024, "weak"),
    "C2": ("16-field mixed 4/8-byte record, 10M records, AoS->SoA", "c2", 10_000_000, "weak"),
    "C3": ("64-field record, SoA->ODS hybrid (128-byte cluster cap), 50M records", "c3", 50_000_000, "weak"),
    "C3R": ("64-field record, SoA->ODS hybrid of the seeded random program (SURVEY 8(d)), 50M records", "c3r",
            50_000_000, "weak"),
    "C4": ("Medical 9x fp32, PDL chain AoS->AoSV->SoA->AoS over 2 GiB of records", "c4", (2 ** 31) // 36, "weak"),
    "C4M": ("Medical 9x fp32, the paper's remap edge AoSV->SoA as a moved subset (adha_remap_regions: the six "
            "unchanged singleton regions aliased, only {V1,V2,V3} move), 2 GiB of records", "c4m", (2 ** 31) // 36,
            "weak"),
    "C5": ("8 GiB mixed-width record array AoS->SoA, sharded across GPUs", "c2", (2 ** 33) // 80, "strong"),
    "P1": ("Medical 256^3 voxels x 9 fp32: AoS->AoSV->SoA", "p1", 256 ** 3, "weak"),
    "P2": ("K-Means 2^23 points x 32 fp32: SoA->4xAoS8->AoS", "p2", 2 ** 23, "weak"),
}


def golden(name):
    """A committed planner-input fixture (tests/golden/*.json): program / arch documents only."""
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        return json.load(fh)


def c3_labels(program="c3_program.json", section="c3"):
    import paper_1407_4859_b200 as A
    layout = A.plan_ods(golden(program), golden("b200_arch.json"), section, "b200")
    names = [f"f{i}" for i in range(64)]
    from adha_inputs import config_widths
    return A.Layout.from_string(layout, names, config_widths(64)).cluster_of, layout


def chain_for(kind):
    """(widths, [label lists along the chain]) of a workload."""
    from adha_inputs import config_widths
    if kind == "xyz":
        return [4, 4, 4], [[0, 0, 0], [0, 1, 2], [0, 0, 0]]
    if kind == "c2":
        w = config_widths(16)
        return w, [[0] * 16, list(range(16))]
    if kind == "c3":
        w = config_widths(64)
        return w, [list(range(64)), c3_labels()[0]]
    if kind == "c3r":      # the seeded random program variant (tests/golden/c3_random_program.json)
        w = config_widths(64)
        return w, [list(range(64)), c3_labels("c3_random_program.json", "c3r")[0]]
    if kind == "c4":
        return [4] * 9, [[0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9)), [0] * 9]
    if kind == "c4m":
        return [4] * 9, [[0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))]
    if kind == "p1":
        return [4] * 9, [[0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))]
    if kind == "p2":
        return [4] * 32, [list(range(32)), [i // 8 for i in range(32)], [0] * 32]
    raise ValueError(kind)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    """dram read+write bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get(config)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled every ~2 ms through NVML while
    running, so that a timed region of a few ms still gets samples; nvidia-smi (100 ms) if NVML
    is unavailable."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap", "hw_power_brake")

    def __init__(self, device_index, period_s=0.002):
        self.dev = device_index
        self.period = period_s
        self.samples = []          # (sm_mhz, power_w, set(reasons))
        self.stop_ev = threading.Event()
        self.max_mhz = None
        self.source = None
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.dev)
            bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def _run_nvml(self, nv, h):
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap,
                "hw_power_brake": nv.nvmlClocksEventReasonHwPowerBrakeSlowdown}
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), pw, {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            time.sleep(self.period)

    def _run_smi(self):
        q = ("clocks.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
             "clocks_event_reasons.hw_power_brake_slowdown")
        p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                              "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        for ln in p.stdout:
            if self.stop_ev.is_set():
                break
            parts = [x.strip() for x in ln.split(",")]
            try:
                self.samples.append((float(parts[0]), float(parts[1]),
                                     {n for n, v in zip(self.NAMES, parts[2:7]) if v.lower() == "active"}))
            except (ValueError, IndexError):
                continue
        p.terminate()

    def start(self):
        try:
            nv, h = self._nvml_handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.source = "nvml, 2 ms"
            self.t = threading.Thread(target=self._run_nvml, args=(nv, h), daemon=True)
        except Exception:
            self.source = "nvidia-smi, 100 ms"
            self.t = threading.Thread(target=self._run_smi, daemon=True)
        self.t.start()

    def count(self):
        return len(self.samples)

    def stop(self):
        self.stop_ev.set()
        if self.t is not None:
            self.t.join(timeout=5)
        if not self.samples:
            return None
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples])
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "sm_min_mhz": min(sm),
                "power_w_median": statistics.median(x[1] for x in self.samples),
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


def oracle_rate(widths, chain, sample_records, seconds, threads):
    """Oracle GB/s (read+write payload) on a sample of the workload, as it stands."""
    import numpy as np
    from adha_inputs import random_bytes
    from oracle import remap as O
    bufs = []
    for k, lab in enumerate(chain):
        nb = O.layout_bytes(widths, lab, sample_records)
        bufs.append(random_bytes(1407 + k, nb) if k == 0 else np.zeros(nb, np.uint8))
    R = sum(widths)
    done = 0
    t0 = time.perf_counter()
    while True:
        for k in range(len(chain) - 1):
            O.remap(bufs[k], chain[k], bufs[k + 1], chain[k + 1], widths, sample_records, threads=threads)
            done += 2 * sample_records * R
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el / 1e9, el


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def planner_times():
    """Host planner cost, off the timed path: the C++ ODS of the C3 program
    (64 fields, 2016 pairs, cap 128 B) and the C++ PDL of the Medical fixture (7 sections x 2
    devices, 56 run nodes); median of 20 calls each, in ms, with the JSON passed as text."""
    import paper_1407_4859_b200 as A

    def med(fn):
        ts = []
        for _ in range(20):
            a = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - a) * 1e3)
        return statistics.median(ts)
    c3p, b200 = json.dumps(golden("c3_program.json")), json.dumps(golden("b200_arch.json"))
    mp, ma, mprof = (json.dumps(golden(x)) for x in ("medical_program.json", "medical_arch.json",
                                                      "medical_profile.json"))
    return {"ods_c3_ms": med(lambda: A.plan_ods(c3p, b200, "c3", "b200")),
            "pdl_medical_ms": med(lambda: A.plan_pdl(mp, ma, mprof)),
            "note": "C++ planner in libadha, host only, off the timed path"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    if rank != 0:
        return 0
    name = args.config
    desc, kind, n_total, scaling = CONFIGS[name]
    widths, chain = chain_for(kind)
    R = sum(widths)
    n = n_total if scaling == "weak" else n_total // max(world, 1)
    sample = min(n, 1 << 20)
    cores = host_cores()
    from oracle import remap as O
    import numpy as np
    from adha_inputs import random_bytes
    bufs = [random_bytes(1407, O.layout_bytes(widths, chain[0], sample))] + \
           [np.zeros(O.layout_bytes(widths, lab, sample), np.uint8) for lab in chain[1:]]

    def step():
        for k in range(len(chain) - 1):
            O.remap(bufs[k], chain[k], bufs[k + 1], chain[k + 1], widths, sample, threads=cores)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    bytes_step = 2 * sample * R * (len(chain) - 1)
    gbs = bytes_step * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": "remap GB/s (read+write)", "value": gbs, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded random bytes)",
        "config": {"workload": f"{name}: {desc}", "records_per_step": sample, "record_bytes": R,
                   "note": "CPU oracle (oracle/remap_oracle.c, plain per-record per-field memcpy) on a bounded "
                           "sample of the workload; no GPU involved"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {sample} records of {name} per step", "cpu_model": cpu_model()},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------------- in-place arm

def run_inplace(args, rank, world, local, share):
    """--inplace: the same workload remapped IN PLACE (adha_remap_inplace, NEXT N1): one buffer of
    max(bytes) per rank instead of one per layout.  A step runs every hop of the config's chain;
    odd steps run the chain backwards, so each step remaps real contents.  `value` counts the
    remap's algorithmic bytes (2 N R per hop, like the out-of-place line); `roofline` is the whole
    in-place step (tile + cycle kernels) against the plans' device traffic."""
    import torch
    import torch.distributed as dist
    import paper_1407_4859_b200 as A
    from paper_1407_4859_b200.sharding import shard_for, max_over_ranks, aggregate_gbs
    from adha_inputs import fill_random_device, SEED_BASE

    dev = torch.device("cuda", local)
    name = args.config
    desc, kind, n_cfg, scaling = CONFIGS[name]
    widths, chain = chain_for(kind)
    R = sum(widths)
    n_total, lo, hi = shard_for(n_cfg, world, rank, scaling)
    n = hi - lo
    lays = [A.Layout(widths, lab) for lab in chain]
    t_plan = time.perf_counter()
    fwd = [A.InplacePlan(lays[k], lays[k + 1], n) for k in range(len(lays) - 1)]
    bwd = [A.InplacePlan(lays[k + 1], lays[k], n) for k in reversed(range(len(lays) - 1))]
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    buf = torch.empty(max(max(p.buffer_bytes for p in fwd + bwd), 256), dtype=torch.uint8, device=dev)
    fill_random_device(buf, SEED_BASE + 1 + rank)
    for p in fwd + bwd:
        p.upload()
    stream = torch.cuda.current_stream(dev)
    hops = len(fwd)
    parity = [0]

    def step():
        for p in (fwd if parity[0] == 0 else bwd):
            A.remap_inplace(buf, p)
        parity[0] ^= 1

    def barrier():
        if world > 1:
            dist.barrier() if share else dist.barrier(device_ids=[local])

    def launches(p):
        d = p.describe()
        return (2 * (d["tail_records"] > 0) + (d["pre_clusters"] > 0) + (d["post_clusters"] > 0)
                + 2 * (d["segments"] > 0))
    for _ in range(max(args.warmup, 3) + (max(args.warmup, 3) % 2)):   # even: the buffer is back in chain[0]
        step()
    torch.cuda.synchronize(dev)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.005)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    ms_total = t0.elapsed_time(t1)
    ms_max = max_over_ranks(ms_total, dev)
    value = aggregate_gbs(n_total, R, hops, args.steps, ms_max)
    n_f, n_b = (args.steps + 1) // 2, args.steps // 2
    traffic_rank = (n_f * sum(p.describe()["traffic_bytes"] for p in fwd)
                    + n_b * sum(p.describe()["traffic_bytes"] for p in bwd))
    n_launch = n_f * sum(launches(p) for p in fwd) + n_b * sum(launches(p) for p in bwd)
    peak, peak_src = measured_peak()
    achieved = traffic_rank / (ms_total * 1e-3) / 1e9

    # end to end through the public API: pinned host records in, in-place remap(s), host records out
    e2e = None
    if not args.no_e2e and n > 0:
        nb0, nbl = lays[0].nbytes(n), lays[-1].nbytes(n)
        h_in = torch.empty(nb0, dtype=torch.uint8).pin_memory()
        h_in.copy_(buf[:nb0].cpu())
        h_out = torch.empty(nbl, dtype=torch.uint8).pin_memory()

        def e2e_step():
            buf[:nb0].copy_(h_in, non_blocking=True)
            for p in fwd:
                A.remap_inplace(buf, p)
            h_out.copy_(buf[:nbl], non_blocking=True)
        e2e_steps = max(3, min(args.steps, 10))
        e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": aggregate_gbs(n_total, R, hops, e2e_steps, e_ms), "unit": "GB/s",
               "h2d_bytes_per_step": nb0, "d2h_bytes_per_step": nbl,
               "api": "H2D copy + adha_remap_inplace x%d + D2H copy" % hops, "ms_per_step": e_ms / e2e_steps}

    if rank == 0:
        line = {
            "metric": "remap GB/s (read+write)", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded random bytes generated on the device)", "impl": "adha-inplace",
            "config": {
                "workload": f"{name} in place: {desc}", "n_records_total": n_total, "n_records_per_rank": n,
                "record_bytes": R, "remaps_per_step": hops, "layouts": [l.to_string() for l in lays],
                "direction": "chain forwards on even steps, backwards on odd steps",
                "buffer_bytes_per_rank": buf.numel(),
                "out_of_place_buffers_bytes_per_rank": sum(l.nbytes(n) for l in lays),
                "workspace_bytes_per_rank": sum(p.workspace_bytes for p in fwd + bwd),
                "plans": [p.describe() for p in fwd],
                "host_plan_ms": plan_ms,
                "host_plans": len(fwd + bwd),
                "host_plan_ms_per_plan": plan_ms / len(fwd + bwd),
                "l2": "inputs larger than L2; no flush" if 2 * n * R > (252 << 20) else "inputs fit in L2 (latency-bound)",
                "parallelism": f"shard by contiguous record range over {world} GPU(s), no data-path collective",
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": ncu_traffic(name + "_inplace"), "traffic_unit": "bytes per step (ncu, all in-place kernels)",
                         "peak_source": peak_src,
                         "kernel": "whole in-place step (ip_tile_kernel + ip_cycle kernels), plan traffic_bytes",
                         "algorithmic_bytes_per_step": traffic_rank / args.steps, "avg_step_ms": ms_total / args.steps},
            "gpu_launches": n_launch, "clocks": clk, "e2e": e2e, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------------------- adha arm

def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn_ranks(n):
    """`--gpus N` without torchrun: re-launch this script as N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line.  Exit code: the launcher's."""
    if os.environ.get("ADHA_BENCH_SHARE_GPU") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="adha", choices=["adha", "reference"])
    ap.add_argument("--inplace", action="store_true",
                    help="remap in place (adha_remap_inplace): one buffer of max(bytes) per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-copy-ref", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: when a step moves < 256 MB, i.e. launch-bound)")
    ap.add_argument("--soak-s", type=float, default=0.0,
                    help="untimed load before the timed region (0: burst regime, like the burst copy peak)")
    ap.add_argument("--sustained-s", type=float, default=3.0,
                    help="after the main measurement: this long untimed under load, then K steps timed again "
                         "(power-capped sustained regime, reported as `sustained`; 0 disables)")
    args = ap.parse_args()

    if args.gpus < 1:
        print("bench.py: --gpus must be >= 1", file=sys.stderr)
        return 2
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            return run_reference(args, 0, args.gpus)     # the CPU oracle: rank 0's work only
        return spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    # ADHA_BENCH_SHARE_GPU=1 (test only): every rank on cuda:0 with a gloo group, to exercise the
    # multi-rank code path on a one-GPU box (the ranks' kernels never wait on one another)
    share = os.environ.get("ADHA_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    if args.inplace:
        return run_inplace(args, rank, world, local, share)

    import paper_1407_4859_b200 as A
    from paper_1407_4859_b200.sharding import shard_for, max_over_ranks, aggregate_gbs
    from adha_inputs import fill_random_device, SEED_BASE

    name = args.config
    desc, kind, n_cfg, scaling = CONFIGS[name]
    widths, chain = chain_for(kind)
    R = sum(widths)
    # shard by contiguous record range: weak -> world * n_cfg records in total, strong -> n_cfg in total
    n_total, lo, hi = shard_for(n_cfg, world, rank, scaling)
    n = hi - lo
    layouts = [A.Layout(widths, lab) for lab in chain]
    plan = A.plan_describe(layouts[0], layouts[1])
    moved = kind == "c4m"          # the remap edge as a moved subset (adha_remap_regions, NEXT N1)
    n_remaps = len(chain) - 1
    if moved:
        # dst regions of identity components alias the src regions (nothing moves there); the other
        # dst clusters get their own regions in one buffer; the metric counts the moved bytes
        L0, L1 = layouts
        keep_src = {c["src_clusters"][0]: c["dst_clusters"][0] for c in plan["components"] if c["identity"]}
        keep_dst = {d: s_ for s_, d in keep_src.items()}
        R_moved = sum(c["R"] for c in plan["components"] if not c["identity"])
        co0, co1 = L0.cluster_of, L1.cluster_of
        src_off = [L0.field_address(co0.index(c), n)[0] for c in range(L0.n_clusters)]
        new_c = [c for c in range(L1.n_clusters) if c not in keep_dst]
        new_bytes = [-(-n * sum(w for w, cc in zip(widths, co1) if cc == c) // 256) * 256 for c in new_c]
        bufs = [torch.empty(max(L0.nbytes(n), 1), dtype=torch.uint8, device=dev),
                torch.empty(max(sum(new_bytes), 1), dtype=torch.uint8, device=dev)]
        fill_random_device(bufs[0], SEED_BASE + 1 + rank)
        bufs[1].fill_(0xA5)
        base0 = bufs[0].data_ptr()
        src_regions = [base0 + o for o in src_off]
        dst_regions, acc = [0] * L1.n_clusters, 0
        for c, nb in zip(new_c, new_bytes):
            dst_regions[c] = bufs[1].data_ptr() + acc
            acc += nb
        for d, s_ in keep_dst.items():
            dst_regions[d] = src_regions[s_]
    else:
        R_moved = R
        bufs = [torch.empty(max(l.nbytes(n), 1), dtype=torch.uint8, device=dev) for l in layouts]
        fill_random_device(bufs[0], SEED_BASE + 1 + rank)
        for b in bufs[1:]:
            b.fill_(0xA5)
    stream = torch.cuda.current_stream(dev)
    bytes_step_rank = 2 * n * R_moved * n_remaps

    def step_direct():
        if moved:
            A.remap_regions(src_regions, layouts[0], dst_regions, layouts[1], n, stream=None)
        elif n_remaps == 1:
            A.remap(bufs[0], layouts[0], bufs[1], layouts[1], n, stream=None)       # torch's current stream
        else:       # a PDL chain: adha_remap_chain (one launch for latency-bound chains like C1)
            A.remap_chain(bufs, layouts, n, stream=None)

    use_graph = args.graph == "on" or (args.graph == "auto" and bytes_step_rank < (256 << 20))
    step = step_direct
    if use_graph:
        # launch-bound step: capture the remap launches once, replay the graph (same kernels, same args)
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for _ in range(3):
                step_direct()
        stream.wait_stream(side)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_direct()
        # launch-bound steps are also captured GRAPH_STEPS at a time, so the timed loop pays one
        # graph launch per GRAPH_STEPS steps (every step still runs its full remap(s))
        graph_n = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_n):
            for _ in range(GRAPH_STEPS):
                step_direct()

        def step():
            graph.replay()

    def run_steps(k):
        """k steps back to back: the multi-step graph where it applies, single steps otherwise."""
        if use_graph:
            for _ in range(k // GRAPH_STEPS):
                graph_n.replay()
            for _ in range(k % GRAPH_STEPS):
                graph.replay()
        else:
            for _ in range(k):
                step()

    def barrier():
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    t_end = time.perf_counter() + args.soak_s
    while time.perf_counter() < t_end:              # optional untimed soak (default 0: burst regime)
        for _ in range(10):
            step()
        torch.cuda.synchronize(dev)

    barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)                    # samples DURING the timed region
    clocks.start()
    time.sleep(0.005)
    w0 = time.perf_counter()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    run_steps(args.steps)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    wall_ms = (time.perf_counter() - w0) * 1e3     # barrier-to-barrier host wall time (context only)
    n_in_region = clocks.count()
    extend_t = time.perf_counter() + 0.5
    while clocks.count() < 5 and time.perf_counter() < extend_t:   # region too short for 5 samples:
        for _ in range(10):                                        # keep the same load on, untimed
            step()
        torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if clk is not None:
        clk["samples_in_timed_region"] = n_in_region
    ms_total = t0.elapsed_time(t1)
    ms_max = max_over_ranks(ms_total, dev)
    wall_max = max_over_ranks(wall_ms, dev)
    value = aggregate_gbs(n_total, R_moved, n_remaps, args.steps, ms_max)

    # per-step spread, measured AFTER the timed region with an event pair around each step
    # (not part of `value`; the per-step events would add their own gaps inside the timed loop)
    reps = []
    for _ in range(min(args.steps, 20)):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        reps.append((a, b))
    torch.cuda.synchronize(dev)
    rep_ms = sorted(a.elapsed_time(b) for a, b in reps)

    # same-run torch copy_ of the same traffic (N*R bytes read + N*R written): the box's copy ceiling now
    copy_gbs = None
    ca = cb = None
    if n > 0 and not args.no_copy_ref:
        ca = torch.empty(n * R_moved, dtype=torch.uint8, device=dev)
        cb = torch.empty_like(ca)
        for _ in range(3):
            cb.copy_(ca)
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(args.steps):
            cb.copy_(ca)
        c1.record(stream)
        torch.cuda.synchronize(dev)
        copy_gbs = 2 * n * R_moved * args.steps / (c0.elapsed_time(c1) * 1e-3) / 1e9

    def sustained_leg(fn, bytes_per_call):
        """fn back to back for --sustained-s seconds (untimed; the board reaches its power-capped
        steady state), then K calls timed with events while NVML samples the clocks."""
        t_end = time.perf_counter() + args.sustained_s
        while time.perf_counter() < t_end:
            for _ in range(10):
                fn()
            torch.cuda.synchronize(dev)
        barrier()
        cs = ClockSampler(local)
        cs.start()
        time.sleep(0.005)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if fn is step:
            run_steps(args.steps)
        else:
            for _ in range(args.steps):
                fn()
        b.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = max_over_ranks(a.elapsed_time(b), dev)
        return bytes_per_call * args.steps * world / (ms * 1e-3) / 1e9, cs.stop()

    sustained = None
    if args.sustained_s > 0 and n > 0:
        v_s, clk_s = sustained_leg(step, 2 * n * R_moved * n_remaps)
        sustained = {"value": v_s, "unit": "GB/s", "clocks": clk_s,
                     "note": f"after {args.sustained_s:.1f} s of untimed load (board power cap engaged); "
                             "K steps timed with events, max over ranks"}
        if ca is not None:
            c_s, cclk_s = sustained_leg(lambda: cb.copy_(ca), 2 * n * R_moved)
            sustained["copy_gbs"] = c_s / world
            sustained["copy_clocks"] = cclk_s
    del ca, cb

    # roofline of the dominant kernel (the remap kernel is the only kernel in the step)
    peak, peak_src = measured_peak()
    # launches per step: one per remap, except a chain of latency-bound hops, which
    # adha_remap_chain runs as ONE fused launch (remap.cu chain_small: every hop <= ADHA_SMALL_BYTES,
    # <= 16 fields, <= 4 hops, packed layouts, disjoint buffers -- all true for C1)
    # routing of adha_remap_chain (remap.cu): one fused launch (tiny chains, or large chains in the
    # tiled kernel's chain mode) or one remap per hop; a single remap takes the direct kernel at
    # payloads <= the plan's direct_bytes
    route, launches_per_step = (A.remap_chain_route(layouts, n) if n_remaps > 1 and not moved
                                else ("single", 1))
    direct = route in ("single", "per_hop") and n * R <= plan["direct_bytes"]
    kernel_name = ("remap_chain_small_kernel (fused chain of latency-bound hops)" if route == "fused_small"
                   else "remap_tiled_kernel in chain mode (all hops in one launch; each intermediate "
                        "read back from L2 while it is written to HBM)" if route == "fused_tiled"
                   else "remap_naive_kernel (direct path for remaps <= the plan's direct_bytes)" if direct
                   else "remap_tiled_kernel")
    # the step is those back-to-back launches and nothing else, so the kernel's average launch
    # duration is this rank's event time over the K steps / (K * launches per step)
    avg_launch_ms = ms_total / (args.steps * launches_per_step)
    # algorithmic HBM bytes per launch: 2 N R per remap; the fused tiled chain reads the src once and
    # writes every intermediate and the dst once ((H + 1) N R), its intermediates come back from L2
    bytes_per_launch = ((n_remaps + 1) * n * R_moved if route == "fused_tiled"
                        else 2 * n * R_moved * n_remaps // launches_per_step)
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    traffic = ncu_traffic(name)

    # end-to-end through the public API with host buffers (pinned), H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e and n > 0:
        h_src = torch.empty(layouts[0].nbytes(n), dtype=torch.uint8).pin_memory()
        h_src.copy_(bufs[0].cpu())
        h_out = torch.empty(bufs[1].numel() if moved else layouts[-1].nbytes(n), dtype=torch.uint8).pin_memory()
        scratch = torch.empty(min(1 << 30, max(64 << 20, 2 * (layouts[0].nbytes(n) + layouts[-1].nbytes(n)))),
                              dtype=torch.uint8, device=dev)
        if moved:   # host AoSV in -> moved-subset remap -> the new {V1},{V2},{V3} regions out
            def e2e_step():
                bufs[0].copy_(h_src, non_blocking=True)
                step_direct()
                h_out.copy_(bufs[1], non_blocking=True)
        elif n_remaps == 1:
            def e2e_step():
                A.remap_host(h_src, layouts[0], h_out, layouts[1], n, scratch, stream=stream)
        else:       # a chain: host in -> device chain -> host out
            def e2e_step():
                bufs[0].copy_(h_src, non_blocking=True)
                step_direct()
                h_out.copy_(bufs[-1], non_blocking=True)
        e2e_steps = max(3, min(args.steps, 10))
        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1), dev)
        e2e = {"value": aggregate_gbs(n_total, R_moved, n_remaps, e2e_steps, e_ms), "unit": "GB/s",
               "h2d_bytes_per_step": h_src.numel(), "d2h_bytes_per_step": h_out.numel(),
               "api": ("H2D copy + adha_remap_regions + D2H copy of the new regions" if moved
                       else "adha_remap_host" if n_remaps == 1
                       else "H2D copy + adha_remap x%d + D2H copy" % n_remaps),
               "ms_per_step": e_ms / e2e_steps}
        del h_src, h_out, scratch

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        sample = min(n, 1 << 20)
        v_all, s_all = oracle_rate(widths, chain, sample, 6.0, cores)
        v_1, s_1 = oracle_rate(widths, chain, sample, 4.0, 1)
        cpu = {"value": v_all, "unit": "GB/s", "cores": cores, "kind": "oracle",
               "sample": f"first {sample} records of {name}, repeated for {s_all:.1f} s "
                         f"(oracle/remap_oracle.c, record-range split over {cores} threads)"
                         + ("; the oracle remaps every field (no aliasing), GB/s of the bytes it moves"
                            if moved else ""),
               "single_thread_value": v_1, "cpu_model": cpu_model()}

    if rank == 0:
        line = {
            "metric": "remap GB/s (read+write)", "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded random bytes generated on the device)",
            "config": {
                "workload": f"{name}: {desc}", "n_records_total": n_total, "n_records_per_rank": n,
                "record_bytes": R, "remaps_per_step": n_remaps,
                "moved_bytes_per_record": R_moved,
                "layouts": [l.to_string() for l in layouts],
                "bytes_per_step_total": 2 * n_total * R_moved * n_remaps,
                "l2": (f"inputs larger than L2 ({2 * n * R_moved / 1e9:.2f} GB moved per remap per GPU vs 126 MB L2); "
                       "no flush" if 2 * n * R_moved > (252 << 20) else
                       f"inputs fit in L2 ({2 * n * R_moved} B per remap; no flush): latency-bound config, not a "
                       "bandwidth claim"),
                "timing_regime": ("burst: timed right after the warm-up, like the burst copy peak"
                                  if args.soak_s <= 0 else f"after a {args.soak_s:.1f} s untimed soak"),
                "parallelism": f"shard by contiguous record range over {world} GPU(s), no data-path collective",
                "kernel": {k: plan[k] for k in ("tiled", "unit", "T", "s_in", "s_out", "smem_bytes", "matched")},
                "chain_route": route,
                "cuda_graph": use_graph,
                "graph_steps_per_launch": GRAPH_STEPS if use_graph else None,
            },
            "records_per_s": n_total * n_remaps * args.steps / (ms_max * 1e-3) / max(n_remaps, 1),
            "pct_of_spec_8000": value / world / 8000.0 * 100.0,
            "same_run_copy_gbs_per_gpu": copy_gbs,
            "frac_of_same_run_copy": (value / world / copy_gbs) if copy_gbs else None,
            "speedup_vs_oracle": ({"all_cores": value / cpu["value"], "single_thread": value / cpu["single_thread_value"],
                                   "paper_context": "PAPER.md:16 reports up to 6.92x from layout choice alone on "
                                                    "X5660 + M2050 (a different quantity; context only)"}
                                  if cpu else None),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         "kernel": kernel_name,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "algorithmic_bytes_note": ("(H+1) N R: the src read once, every intermediate and the dst "
                                                    "written once to HBM; the metric's 2 N R per hop counts the "
                                                    "intermediates' reads too, which come from L2"
                                                    if route == "fused_tiled" else "2 N R per remap"),
                         "avg_launch_ms": avg_launch_ms},
            "sustained": sustained,
            "planner": planner_times(),
            "step_ms_spread": {"median": statistics.median(rep_ms), "min": rep_ms[0], "max": rep_ms[-1],
                               "reps": len(rep_ms), "note": "per-step events after the timed region, rank 0"},
            "wall_ms_timed_region": wall_max,
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
