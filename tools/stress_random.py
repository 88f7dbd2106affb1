"""Randomised GPU stress: many random layout pairs (packed, C-aligned, AoSoA blocks), random N
(tile boundaries, ragged tails, tiny and large), both write-back modes forced and automatic, the
tiled kernel forced (ADHA_SMALL_BYTES=0) -- every result compared byte for byte with the CPU
oracle.  Not part of the test suite (minutes of run time); prints the number of cases and the
first failure.   usage: python tools/stress_random.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import field_columns  # noqa: E402
from oracle import remap as O  # noqa: E402

CASES = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 14074859)
os.environ["ADHA_SMALL_BYTES"] = "0"
SENT = 0xA5
fails = 0
for case in range(CASES):
    F = int(rng.integers(1, 24))
    widths = [int(x) for x in rng.choice([1, 2, 3, 4, 4, 4, 8, 8, 12, 16], size=F)]

    def rand_layout():
        labels = [int(x) for x in rng.integers(0, max(1, F // int(rng.integers(1, 4))), size=F)]
        blocks = None
        if rng.random() < 0.25:
            per = {c: int(rng.choice([1, 2, 4, 8, 16, 32])) for c in set(labels)}
            blocks = [per[c] for c in labels]
        return labels, blocks, bool(rng.random() < 0.25)

    (ls, bs, als), (ld, bd, ald) = rand_layout(), rand_layout()
    n = int(rng.choice([1, 31, 32, 33, 1000, 4095, 4097, int(rng.integers(1, 300_000))]))
    mode = str(rng.choice(["auto", "tma", "stg"]))
    if mode == "auto":
        os.environ.pop("ADHA_COPYOUT", None)
    else:
        os.environ["ADHA_COPYOUT"] = mode
    cols = field_columns(case, n, widths)
    src = O.pack_ex(cols, widths, ls, n, bs, als, fill=0x3C)
    Ls = A.Layout(widths, ls, blocks=bs, aligned=als)
    Ld = A.Layout(widths, ld, blocks=bd, aligned=ald)
    d_src = torch.from_numpy(src).cuda() if src.size else torch.zeros(1, dtype=torch.uint8, device="cuda")
    d_dst = torch.full((max(1, Ld.nbytes(n)),), SENT, dtype=torch.uint8, device="cuda")
    A.remap(d_src, Ls, d_dst, Ld, n)
    torch.cuda.synchronize()
    exp = np.full(O.layout_bytes_ex(widths, ld, n, bd, ald), SENT, np.uint8)
    O.remap_ex(src, ls, exp, ld, widths, n, bs, als, bd, ald)
    got = d_dst.cpu().numpy()[: exp.size]
    if not np.array_equal(got, exp):
        fails += 1
        bad = np.nonzero(got != exp)[0]
        print(f"FAIL case {case}: widths={widths} ls={ls} bs={bs} als={als} ld={ld} bd={bd} ald={ald} n={n} "
              f"mode={mode} plan={ {k: v for k, v in A.plan_describe(Ls, Ld).items() if not isinstance(v, (list, dict))} } "
              f"bad={bad.size} first={bad[:8]}", flush=True)
        if fails >= 3:
            break
print(f"{CASES} random cases, {fails} failures")
