"""Randomised GPU stress of the in-place remap (adha_remap_inplace): many random packed layout
pairs (widths from 1 to 16 bytes, so u = 1, 2, 4, 8 and 16 all occur), random N (tile boundaries,
ragged tails, tiny and large; up to MAX_N), each plan run forwards and then backwards on the same buffer.
Every dst payload byte is compared with the CPU oracle's out-of-place remap, and the round trip
with the original records.  Not part of the test suite (minutes of run time); prints the number
of cases and the first failure.   usage: python tools/stress_inplace.py [cases] [seed] [max_n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import field_columns  # noqa: E402
from oracle import remap as O  # noqa: E402

CASES = int(sys.argv[1]) if len(sys.argv) > 1 else 300
# the slot-permutation kernels at every size (small buffers would otherwise take the staged mode,
# an out-of-place remap through the workspace; ADHA_INPLACE_STAGED_BYTES=-1 keeps the default)
if os.environ.get("ADHA_INPLACE_STAGED_BYTES") != "-1":
    os.environ["ADHA_INPLACE_STAGED_BYTES"] = "0"
else:
    os.environ.pop("ADHA_INPLACE_STAGED_BYTES")
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 14074859)
MAX_N = int(sys.argv[3]) if len(sys.argv) > 3 else 400_000
fails = 0
stats = {}
for case in range(CASES):
    F = int(rng.integers(1, 40))
    pool = [rng.choice([1, 2, 3, 4, 8, 12, 16]), rng.choice([4, 8, 16]), 4]
    widths = [int(x) for x in rng.choice(pool, size=F)]

    def rand_labels():
        return [int(x) for x in rng.integers(0, max(1, F // int(rng.integers(1, 5))), size=F)]

    ls, ld = rand_labels(), rand_labels()
    n = int(rng.choice([1, 63, 64, 65, 255, 256, 257, 1000, 4097, int(rng.integers(1, MAX_N))]))
    Ls, Ld = A.Layout(widths, ls), A.Layout(widths, ld)
    try:
        fwd, bwd = A.InplacePlan(Ls, Ld, n), A.InplacePlan(Ld, Ls, n)
    except A.AdhaError as e:        # e.g. a record too wide for a tile: counted, not a failure
        stats[e.name] = stats.get(e.name, 0) + 1
        continue
    d = fwd.describe()
    stats[f"u{d['unit']}"] = stats.get(f"u{d['unit']}", 0) + 1
    cols = field_columns(case, n, widths)
    src = O.pack(cols, widths, ls, n, fill=0x3C)
    buf = torch.full((max(fwd.buffer_bytes, bwd.buffer_bytes, 256),), 0x5A, dtype=torch.uint8, device="cuda")
    buf[: src.size].copy_(torch.from_numpy(src))
    A.remap_inplace(buf, fwd)
    torch.cuda.synchronize()
    got = buf.cpu().numpy()
    exp = np.zeros(O.layout_bytes(widths, ld, n), np.uint8)
    O.remap(src, ls, exp, ld, widths, n)
    mask = O.payload_mask(widths, ld, n)
    ok = np.array_equal(got[: exp.size][mask], exp[mask])
    A.remap_inplace(buf, bwd)
    torch.cuda.synchronize()
    back = buf.cpu().numpy()[: src.size]
    mask_s = O.payload_mask(widths, ls, n)
    ok = ok and np.array_equal(back[mask_s], src[mask_s])
    if not ok:
        fails += 1
        if fails == 1:
            print("FIRST FAILURE", {"case": case, "widths": widths, "ls": ls, "ld": ld, "n": n, "plan": d}, flush=True)
print({"cases": CASES, "failures": fails, "by_unit_or_status": stats}, flush=True)
sys.exit(1 if fails else 0)
