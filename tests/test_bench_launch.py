"""bench.py's launch contract on CPU: `--gpus N` without a torchrun environment re-launches the
script as N ranks (torch.distributed.run on 127.0.0.1) and rank 0 reports the world; a
mismatched --gpus / WORLD_SIZE fails loudly instead of silently timing one rank."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       env=e, timeout=300, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    return r.returncode, [json.loads(l) for l in lines], r.stderr


def test_gpus2_self_launches_two_ranks():
    rc, out, err = _run(["--gpus", "2", "--dry-run"])
    assert rc == 0, err
    assert len(out) == 1, out                       # rank 0 alone prints
    line = out[0]
    assert line["n_gpus"] == 2 and line["gpus_flag"] == 2
    ranks = sorted(line["ranks"], key=lambda r: r["rank"])
    assert [(r["rank"], r["world_size"], r["local_rank"]) for r in ranks] == [(0, 2, 0), (1, 2, 1)]


def test_single_rank_default_and_mismatch_rejected():
    rc, out, _ = _run(["--dry-run"])
    assert rc == 0 and out[0]["n_gpus"] == 1
    rc, out, _ = _run(["--gpus", "4", "--dry-run"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc == 2 and "error" in out[0]


def test_reference_arm_line_has_the_contract_keys():
    """`--impl reference` times the oracle on host cores and prints the base contract's line plus
    `impl`, `cpu_baseline` and a zero-copy `e2e` (no GPU work: gpu_launches 0)."""
    rc, out, err = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "cfg2",
                         "--ref-budget", "0.5"])
    assert rc == 0, err
    line = out[-1]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e", "vs_baseline"):
        assert k in line, k
    assert line["impl"] == "reference" and line["gpu_launches"] == 0 and line["n_gpus"] == 1
    assert line["value"] > 0 and line["ms_per_step"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"] == "cfg2"
