"""bench.py's reference arm under torchrun on CPU (world size 2, 127.0.0.1):
rank 0 alone times the oracle and prints exactly one JSON line with the
contract's keys; the other rank exits 0 without work."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reference_arm_torchrun_world2():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_our_arm_json_line_on_the_gpu():
    """Our arm on one B200 (the C2 workload, a short run): one JSON line
    with every key of the driver's contract, the roofline and cpu_baseline
    objects, the e2e object through the host-buffer batch entry, the launch
    count of the timed region (10 frames per step), clocks sampled during it,
    evals counted as active pairs (<= the replicated valid x lights count)."""
    cmd = [sys.executable, "bench.py", "--config", "C2", "--steps", "3", "--warmup", "3", "--e2e-steps", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["scaling"] == "strong"
    assert d["value"] > 1e9 and d["higher_is_better"] is True and d["vs_baseline"] is None
    cf = d["config"]
    assert cf["workload"].startswith("C2") and cf["launches_per_step_per_rank"] == 10
    assert 0 < cf["evals_per_step_per_rank"] <= cf["evals_replicated_per_step_per_rank"]
    assert cf["verified"].startswith("all 10 frames written")
    assert d["gpu_launches"] == 30
    ro = d["roofline"]
    assert ro["bound"] == "alu" and 0 < ro["frac"] < 1 and ro["peak"] > 0
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert abs(ro["mean_launch_ms"] - d["ms_per_step"] / 10) < 1e-6 * d["ms_per_step"] + 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] > 0
    e = d["e2e"]
    assert e["api"].startswith("glint_eval_host_batch") and e["value"] > 0
    assert e["h2d_bytes_per_step"] == cf["pixels_per_step_per_rank"] * 80
    assert e["d2h_bytes_per_step"] == cf["pixels_per_step_per_rank"] * 16
    c = d["clocks"]
    assert isinstance(c["reasons"], list) and "samples" in c
    if c["samples"]:      # a 3-step region is short: NVML may not have sampled it
        assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0
    else:
        assert c["reasons"] == ["nvml_unavailable"]


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["C3", "C2"])
def test_our_arm_two_ranks_one_gpu(config):
    """The N > 1 code path of our arm, functionally, on the one GPU of this
    box: torchrun with 2 ranks, both on cuda:0 (GLINT_BENCH_DEVICE), gloo for
    the control plane (NCCL refuses two ranks on one device). C3 is one frame
    cut into 64-row bands, C2 ten whole frames dealt to 2 ranks; rank 1's
    kernels store its tiles through their tile origins into rank 0's
    IPC-mapped full frames (the fused gather). Rank 0 alone prints one line
    with n_gpus 2; every pixel was written and rank-1 tiles re-evaluated on
    rank 0 are bit-identical. (Timing here is meaningless: two processes share
    one GPU.)"""
    args = ["bench.py", "--gpus", "2", "--config", config, "--steps", "2", "--warmup", "3", "--no-e2e",
            "--no-cpu-baseline"]
    if config == "C3":    # launched as the driver does
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), *args]
    else:                 # bench.py re-executes itself through torchrun (no WORLD_SIZE in the environment)
        cmd = [sys.executable, *args]
    env = dict(os.environ, GLINT_BENCH_BACKEND="gloo", GLINT_BENCH_DEVICE="0")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    cf = d["config"]
    assert "bit-identical" in cf["verified"] and "fused" in cf["gather"]
    assert ("64-row bands" in cf["parallelism"]) == (config == "C3")
    assert d["gpu_launches"] == 2 * cf["tiles_per_step"]
    assert cf["compute_only"]["value"] > 0 and cf["rank0_ms_per_step"] > 0


def test_bench_refuses_a_mismatched_world():
    """--gpus N under a world of another size prints no result line."""
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and not any(ln.startswith("{") for ln in r.stdout.splitlines())
    assert "refusing" in r.stderr
