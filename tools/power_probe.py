"""Sustained power/clock/throughput of the C2 remap vs torch copy_ of the same bytes.

Each variant runs back-to-back for SECONDS while nvidia-smi samples power.draw and clocks.sm
every 50 ms; GB/s is measured with CUDA events over 100-step windows in the second half.
Question: under the board power cap, does the remap draw more power (and so lose SM clock)
than a plain device copy moving the same bytes?
usage: python tools/power_probe.py [SECONDS]
"""
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1407_4859_b200 as A
from adha_inputs import config_widths, fill_random_device

SECONDS = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
N = 10_000_000
w = config_widths(16)
R = sum(w)
La, Ls = A.Layout.aos(w), A.Layout.soa(w)
src = torch.empty(La.nbytes(N), dtype=torch.uint8, device="cuda")
dst = torch.empty(Ls.nbytes(N), dtype=torch.uint8, device="cuda")
fill_random_device(src, 5)
ca = torch.empty(N * R, dtype=torch.uint8, device="cuda")
cb = torch.empty_like(ca)


class Sampler:
    def __init__(self):
        self.rows, self.stop_ev = [], threading.Event()

    def run(self):
        p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks.mem,temperature.gpu",
                              "--format=csv,noheader,nounits", "-i", "0", "-lms", "50"],
                             stdout=subprocess.PIPE, text=True)
        for line in p.stdout:
            if self.stop_ev.is_set():
                break
            try:
                self.rows.append((time.perf_counter(), [float(x) for x in line.split(",")]))
            except ValueError:
                pass
        p.terminate()


def run(name, fn):
    s = Sampler()
    th = threading.Thread(target=s.run, daemon=True)
    th.start()
    time.sleep(0.3)
    t_start = time.perf_counter()
    rates = []
    while time.perf_counter() - t_start < SECONDS:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            fn()
        e1.record()
        e1.synchronize()
        if time.perf_counter() - t_start > SECONDS / 2:
            rates.append(2 * N * R * 100 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    t_end = time.perf_counter()
    s.stop_ev.set()
    th.join(timeout=2)
    late = [v for t, v in s.rows if t_start + SECONDS / 2 <= t <= t_end]
    pw = statistics.mean(v[0] for v in late) if late else float("nan")
    sm = statistics.median(v[1] for v in late) if late else float("nan")
    mem = statistics.median(v[2] for v in late) if late else float("nan")
    temp = max(v[3] for v in late) if late else float("nan")
    gbs = statistics.mean(rates)
    print(f"{name:28s} {gbs:7.0f} GB/s  power {pw:6.1f} W  sm {sm:6.0f} MHz  mem {mem:5.0f} MHz  "
          f"temp {temp:4.0f} C  J/GB {pw / gbs:.4f}", flush=True)
    time.sleep(2.0)          # cool-down between variants


def remap_env(env):
    def fn():
        os.environ.update(env)
        A.remap(src, La, dst, Ls, N)
        for k in env:
            del os.environ[k]
    return fn


variants = [("copy_", lambda: cb.copy_(ca)), ("remap C2", lambda: A.remap(src, La, dst, Ls, N))]
for extra in sys.argv[2:]:              # e.g. ADHA_STAGE_BYTES=40960,ADHA_OUT_BUFFERS=1
    variants.append((f"remap C2 {extra}", remap_env(dict(kv.split("=") for kv in extra.split(",")))))
for _ in range(2):
    for name, fn in variants:
        run(name, fn)
