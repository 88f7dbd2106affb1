"""Drift-cancelled A/B of several env-knob variants (each a set of ADHA_* settings, read by the
library when a plan is compiled or a call is made) over the bench chain edges, in one process.
    python tools/ab_multi.py "A=1,B=2" "A=3" ...      (an empty string is the default variant)
Prints, per edge, the median GB/s of each variant over ROUNDS interleaved rounds."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import fill_random_device  # noqa: E402
import bench  # noqa: E402

ROUNDS = int(os.environ.get("ROUNDS", "5"))
variants = [dict(kv.split("=") for kv in v.split(",") if kv) for v in (sys.argv[1:] or [""])]
edges = []
if os.environ.get("NARROW") == "1":          # the narrow-field / generalised cases of narrow_probe.py
    for name, w in (("g2", [2, 4, 6, 4] * 4), ("g1", [1, 3, 4, 8] * 4), ("b24", [1] * 24 + [8])):
        F = len(w)
        edges.append((name + "a2s", w, [0] * F, list(range(F)), 20_000_000))
        edges.append((name + "s2a", w, list(range(F)), [0] * F, 20_000_000))
for cfg in [c for c in os.environ.get("CFGS", "C2,P1,P2,C4").split(",") if c]:
    desc, kind, n, _ = bench.CONFIGS[cfg]
    widths, chain = bench.chain_for(kind)
    for k in range(len(chain) - 1):
        edges.append((f"{cfg}/{k}", widths, chain[k], chain[k + 1], n))
big = max(max(A.Layout(w, a).nbytes(n), A.Layout(w, b).nbytes(n)) for _, w, a, b, n in edges)
buf_a = torch.empty(big, dtype=torch.uint8, device="cuda")
buf_b = torch.empty(big, dtype=torch.uint8, device="cuda")
fill_random_device(buf_a, 9)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {}
for rnd in range(ROUNDS):
    for name, w, ls, ld, n in edges:
        R = sum(w)
        for vi, env in enumerate(variants):
            saved = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)          # fresh handles: the plan recompiles
            ms = timed(lambda: A.remap(buf_a, Ls, buf_b, Ld, n))
            for k, v in saved.items():
                if v is None:
                    del os.environ[k]
                else:
                    os.environ[k] = v
            res.setdefault((name, vi), []).append(2 * n * R / (ms * 1e-3) / 1e9)
print("variants:", [",".join(f"{k}={v}" for k, v in e.items()) or "default" for e in variants])
for name, *_ in edges:
    print(f"{name:6s} " + "  ".join(f"{statistics.median(res[(name, vi)]):7.0f}" for vi in range(len(variants))))
