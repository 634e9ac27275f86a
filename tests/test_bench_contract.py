"""bench.py's reference arm on CPU (no GPU): the JSON line carries the contract's keys, and
ranks other than 0 print nothing and exit 0."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None):
    env = dict(os.environ)
    env.update(extra_env or {})
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "1"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.strip()]


def test_reference_arm_line():
    lines = _run()
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in out, k
    assert out["value"] > 0 and out["unit"] == "DOF/s" and out["higher_is_better"] is True
    assert out["config"]["dof"] == 816          # 16 leaves x 6^2 interior + 40 edges x 6 (corner-free p = 8)
    cb = out["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == out["value"] and cb["cores"] >= 1
    assert out["e2e"]["value"] == out["value"]
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_root_R_rule_and_flop_model():
    """SURVEY hard part 8: R^1 formed for configs 1-3, skipped for 4-5; the flop model drops exactly
    the root's R^tau product (8 n_tau^2 n3 at the root) when it is skipped."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1812_07167_b200 import inputs
    assert [bench.root_R_default(c) for c in (1, 2, 3, 4, 5)] == [True, True, True, False, False]
    for c in (2, 4):
        cfg = inputs.CONFIGS[c]
        d, n3, n1, ntau = bench.merge_levels(cfg)[0]
        assert d == 0
        assert bench.flop_model(cfg) - bench.flop_model(cfg, root_R=False) == 8.0 * ntau * ntau * n3
