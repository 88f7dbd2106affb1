"""Shared-memory wavefronts of a byte-group plan, simulated on the host for every period phase.

A warp instruction of the byte-group permute has all 32 lanes at the same period q; lane l of
slot m loads the 4-byte word at chunk_smem(c) + off + q * 32 * stride_c.  The bank of that word
moves by 8 * stride_c words per period, so a plan that is conflict-free at q = 0 can conflict at
odd q when clusters of stride 2 (mod 4) and stride 0 (mod 4) share an instruction.  This prints
wavefronts per load / store instruction averaged over q = 0..3 (ideal: 1.0).
usage: python tools/bank_sim.py
"""
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_4859_b200 as A  # noqa: E402


def wavefronts(addrs):
    """32-bit shared accesses: wavefronts = max over banks of distinct word addresses."""
    per_bank = {}
    for a in addrs:
        per_bank.setdefault((a // 4) % 32, set()).add(a // 4)
    return max((len(v) for v in per_bank.values()), default=0)


def simulate(Ls, Ld):
    d = A.plan_describe(Ls, Ld)
    if not d.get("byte_groups"):
        return None
    res = Counter()
    for K in d["components"]:
        if K["identity"]:
            continue
        groups = d["groups"][K["instr_base"]: K["instr_base"] + K["n_instr"]]
        # chunk stagger: 32 B per cluster index inside the component (remap_plan.cpp), keyed by
        # kernel cluster slot (position in src_order / dst_order)
        src_pad = {}
        for i, c in enumerate(K["src_clusters"]):
            src_pad[d["src_order"].index(c)] = 32 * i
        dst_pad = {}
        for i, c in enumerate(K["dst_clusters"]):
            dst_pad[d["dst_order"].index(c)] = 32 * i
        for i0 in range(0, len(groups), 32):
            ins = groups[i0: i0 + 32]
            for q in range(4):
                for m in range(4):
                    addrs = [src_pad[g[14 + m]] + g[10 + m] + q * 32 * d["src_stride"][g[14 + m]]
                             for g in ins if m < g[1]]
                    if addrs:
                        res["ld_instr"] += 1
                        res["ld_wf"] += wavefronts(addrs)
                for o in range(4):
                    addrs = [dst_pad[g[6 + o]] + g[2 + o] + q * 32 * d["dst_stride"][g[6 + o]]
                             for g in ins if o < g[0]]
                    if addrs:
                        res["st_instr"] += 1
                        res["st_wf"] += wavefronts(addrs)
    return res


CASES = {
    "g2 AoS->SoA [2,4,6,4]x4": ([2, 4, 6, 4] * 4, "aos", "soa"),
    "g2 SoA->AoS [2,4,6,4]x4": ([2, 4, 6, 4] * 4, "soa", "aos"),
    "g1 AoS->SoA [1,3,4,8]x4": ([1, 3, 4, 8] * 4, "aos", "soa"),
    "g1 SoA->AoS [1,3,4,8]x4": ([1, 3, 4, 8] * 4, "soa", "aos"),
    "g1 AoS->SoA 24x1+8": ([1] * 24 + [8], "aos", "soa"),
    "g1 SoA->AoS 24x1+8": ([1] * 24 + [8], "soa", "aos"),
    "SoA->aligned AoS {1,4,2,8,4,2}": ([1, 4, 2, 8, 4, 2], "soa", "aligned"),
    "aligned AoS->SoA {1,4,2,8,4,2}": ([1, 4, 2, 8, 4, 2], "aligned", "soa"),
}


def make(w, kind):
    F = len(w)
    if kind == "aos":
        return A.Layout(w, [0] * F)
    if kind == "soa":
        return A.Layout(w, list(range(F)))
    return A.Layout(w, [0] * F, aligned=True)


if __name__ == "__main__":
    for name, (w, a, b) in CASES.items():
        r = simulate(make(w, a), make(w, b))
        if r is None:
            print(f"{name:34s} (not byte-group mode)")
            continue
        print(f"{name:34s} ld {r['ld_wf'] / max(1, r['ld_instr']):5.2f} wf/instr   "
              f"st {r['st_wf'] / max(1, r['st_instr']):5.2f} wf/instr   "
              f"({r['ld_instr'] // 4} ld + {r['st_instr'] // 4} st instr per period)")
