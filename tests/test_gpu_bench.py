"""bench.py on a GPU: the JSON line keeps the driver's contract (keys, units, clocks sampled in the
timed region, roofline, e2e, gpu_launches), and the torchrun multi-rank path (ranks sharing the one
GPU through ADHA_BENCH_SHARE_GPU; their kernels never wait on one another) reports the max over
ranks with weak scaling."""
import json
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline")


def run_bench(args, env=None, torchrun=0):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py")] + args
    if torchrun:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={torchrun}",
               "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py")] + args
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=e)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_c2_contract():
    d = run_bench(["--config", "C2", "--steps", "20", "--warmup", "3", "--sustained-s", "0.3", "--no-cpu-baseline"])
    for k in KEYS:
        assert k in d, k
    assert d["metric"] == "remap GB/s (read+write)" and d["unit"] == "GB/s" and d["dtype"] == "u8"
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C2") and d["vs_baseline"] is None
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] == 20
    assert d["clocks"]["samples"] >= 5 and d["clocks"]["sm_mhz"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 10_000_000 * 80 == d["e2e"]["d2h_bytes_per_step"]
    assert d["sustained"]["value"] > 0 and d["sustained"]["copy_gbs"] > 0
    assert d["value"] > 1000          # a B200 moves well over 1 TB/s through the remap


def test_bench_c1_graph():
    d = run_bench(["--config", "C1", "--steps", "50", "--warmup", "3", "--sustained-s", "0", "--no-cpu-baseline"])
    assert d["config"]["cuda_graph"] is True and d["gpu_launches"] == 50      # fused chain: 1 launch per step
    assert "fit in L2" in d["config"]["l2"]


def test_bench_two_ranks_share_gpu():
    d = run_bench(["--config", "C2", "--gpus", "2", "--steps", "5", "--warmup", "3", "--sustained-s", "0",
                   "--no-e2e", "--no-copy-ref"], env={"ADHA_BENCH_SHARE_GPU": "1"}, torchrun=2)
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["n_records_total"] == 2 * d["config"]["n_records_per_rank"]


def test_bench_default_is_c5_and_gpus_spawns_ranks():
    """No --config: C5 (BASELINE.json's metric, "at 1/2/4/8 B200"), strong-scaled.  `--gpus 2`
    WITHOUT torchrun re-launches bench.py as two ranks (here sharing the one GPU through
    ADHA_BENCH_SHARE_GPU): n_gpus == 2 and the 8 GiB array is split two ways."""
    d = run_bench(["--gpus", "2", "--steps", "5", "--warmup", "3", "--sustained-s", "0", "--no-e2e",
                   "--no-copy-ref"], env={"ADHA_BENCH_SHARE_GPU": "1"})
    assert d["config"]["workload"].startswith("C5") and d["scaling"] == "strong"
    assert d["n_gpus"] == 2
    c = d["config"]
    assert c["n_records_total"] == 2 ** 33 // 80 and c["n_records_per_rank"] == c["n_records_total"] // 2
    assert d["roofline"]["kernel"] == "remap_tiled_kernel" and d["value"] > 1000


def test_bench_gpus_mismatch_fails():
    """--gpus N under a launcher with another WORLD_SIZE is an error, not a silent 1-rank run."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3"]
    e = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=e)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_bench_c4m_moved_subset():
    """C4M: the Medical AoSV->SoA edge through adha_remap_regions; 12 of 36 bytes per record move
    (SPEC.md:221), and the line counts exactly those bytes."""
    d = run_bench(["--config", "C4M", "--steps", "10", "--warmup", "3", "--sustained-s", "0",
                   "--no-cpu-baseline"])
    c = d["config"]
    assert c["moved_bytes_per_record"] == 12 and c["record_bytes"] == 36
    assert c["bytes_per_step_total"] == 2 * 12 * (2 ** 31 // 36)
    assert d["roofline"]["algorithmic_bytes_per_launch"] == 2 * 12 * (2 ** 31 // 36)
    assert d["e2e"]["d2h_bytes_per_step"] < d["e2e"]["h2d_bytes_per_step"]
    assert d["value"] > 1000 and d["gpu_launches"] == 10


@pytest.mark.parametrize("cfg", ["C2", "C4"])
def test_bench_inplace_contract(cfg):
    """--inplace: the same contract keys; C4's chain returns to AoS each step, C2 alternates
    direction; the buffer is max(bytes), not the sum."""
    d = run_bench(["--inplace", "--config", cfg, "--steps", "6", "--warmup", "3"])
    for k in KEYS:
        assert k in d, k
    assert d["impl"] == "adha-inplace" and d["value"] > 500
    c = d["config"]
    assert c["buffer_bytes_per_rank"] < c["out_of_place_buffers_bytes_per_rank"]
    assert 0 < d["roofline"]["frac"] < 1.2 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0


def test_bench_inplace_two_ranks_share_gpu():
    d = run_bench(["--inplace", "--gpus", "2", "--steps", "4", "--warmup", "3", "--no-e2e"],
                  env={"ADHA_BENCH_SHARE_GPU": "1"}, torchrun=2)
    assert d["n_gpus"] == 2 and d["impl"] == "adha-inplace"
    assert d["config"]["n_records_total"] == 2 * d["config"]["n_records_per_rank"]
