"""Direct (latency) kernel vs tiled kernel for small and mid-size remaps: GPU time per remap from
CUDA-graph replay (20 remaps per graph, so host launch cost is excluded), for several record
shapes and payload sizes, with ADHA_SMALL_BYTES forcing one path or the other.  Used to place
the direct-path threshold.   usage: python tools/small_path_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1407_4859_b200 as A  # noqa: E402
from adha_inputs import config_widths  # noqa: E402

SHAPES = {
    "C2 AoS->SoA": (config_widths(16), [0] * 16, list(range(16))),
    "C2 SoA->AoS": (config_widths(16), list(range(16)), [0] * 16),
    "Medical AoS->AoSV": ([4] * 9, [0] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6]),
    "K-Means SoA->AoS (32 f)": ([4] * 32, list(range(32)), [0] * 32),
    "C3 SoA->hybrid (64 f)": (config_widths(64), list(range(64)), None),
    "narrow 24x1B+8 AoS->SoA": ([1] * 24 + [8], [0] * 25, list(range(25))),
    "Medical AoSV->SoA": ([4] * 9, [0, 0, 0, 1, 2, 3, 4, 5, 6], list(range(9))),
    "K-Means 4xAoS8->AoS": ([4] * 32, [f // 8 for f in range(32)], [0] * 32),
    "g2 [2,4,6,4]x4 AoS->SoA": ([2, 4, 6, 4] * 4, [0] * 16, list(range(16))),
    "C3 hybrid->SoA (64 f)": (config_widths(64), None, list(range(64))),
}


def graph_us(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / 100


def main():
    import bench
    for name, (w, ls, ld) in SHAPES.items():
        if len(sys.argv) > 1 and name not in sys.argv[1:]:
            continue
        if ld is None:
            ld = bench.c3_labels()[0]
        if ls is None:
            ls = bench.c3_labels()[0]
        R = sum(w)
        Ls, Ld = A.Layout(w, ls), A.Layout(w, ld)
        for payload in (256 << 10, 1 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20, 128 << 20, 512 << 20):
            n = max(1, payload // R)
            src = torch.zeros(Ls.nbytes(n), dtype=torch.uint8, device="cuda")
            dst = torch.zeros(Ld.nbytes(n), dtype=torch.uint8, device="cuda")
            out = {"shape": name, "payload_MB": round(n * R / 2 ** 20, 2),
                   "components": len(A.plan_describe(Ls, Ld)["components"])}
            # tiled: the default plan choice (merged plan up to merge_bytes); tiled_merged: the
            # merged plan at every size; tiled_components: the per-component (large-N) plan;
            # direct: the direct kernel
            for path, env in (("tiled", {"ADHA_SMALL_BYTES": "0"}),
                              ("tiled_merged", {"ADHA_SMALL_BYTES": "0", "ADHA_MERGE_BYTES": str(1 << 40)}),
                              ("tiled_components", {"ADHA_SMALL_BYTES": "0", "ADHA_MERGE_BYTES": "0"}),
                              ("direct", {"ADHA_SMALL_BYTES": str(1 << 40)})):
                for k in ("ADHA_SMALL_BYTES", "ADHA_MERGE_BYTES"):
                    os.environ.pop(k, None)
                os.environ.update(env)
                out[path + "_us"] = round(graph_us(lambda: A.remap(src, Ls, dst, Ld, n)), 2)
            for k in ("ADHA_SMALL_BYTES", "ADHA_MERGE_BYTES"):
                os.environ.pop(k, None)
            out["default_us"] = round(graph_us(lambda: A.remap(src, Ls, dst, Ld, n)), 2)
            print(json.dumps(out), flush=True)
            del src, dst


if __name__ == "__main__":
    main()
