"""CPU check of bench.py's reference arm (the oracle timed on the host): one JSON
line with the contract's keys, on the tiny config (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "tiny", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline",
              "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_flag_spawns_one_process_per_gpu_and_rank0_prints_once():
    """`bench.py --gpus 2` without a launcher re-runs itself under torchrun with
    two ranks (WORLD_SIZE=2); for the reference arm rank 0 alone prints."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--workload", "tiny", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "summands/2"


def test_both_arms_share_the_config_object():
    sys.path.insert(0, ROOT)
    import bench
    for w in bench.WORKLOADS:
        c = bench.bench_config(w, "rand_orth", 1)
        assert c["workload"] == w and c["summands"] >= 1 and c["d"] >= 2
    # the full-shape bond sample of config 5 really has config 5's per-bond shapes
    terms, f_s, f_f = bench.large_bond_sample()
    assert len(terms) == 32
    assert [c.shape for c in terms[0]] == [(144, 256, 64), (64, 256, 64), (64, 256, 1)]
    assert 20 < f_f / f_s < 60
