"""CPU tests of bench.py's host plumbing (no GPU): `--gpus 2` outside
torchrun spawns two ranks through torch.distributed.run, they form a gloo
group, build their sharded plans offline and reduce a max over ranks; rank 0
prints one JSON line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=240):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                       text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("config,mode", [("s5redist", "redistribute"), ("s5local", "local"),
                                         ("s5p2p", "p2p")])
def test_bench_spawns_two_ranks_dry_run(config, mode):
    j = _run(["--gpus", "2", "--config", config, "--dry-run"])
    assert j["dry_run"] is True and j["n_gpus"] == 2 and j["config"] == config
    assert j["max_over_ranks"] == 2.0          # rank 1's value survives the MAX reduction
    assert j["mode"] == mode
    assert j["plan"]["nranks"] == 2
    if config == "s5redist":
        assert j["plan"]["local_in_dims"] == [112, 112, 112, 52]


def test_bench_single_rank_dry_run():
    j = _run(["--dry-run"])
    assert j["n_gpus"] == 1 and j["plan"]["kernel"] == "tiled2d"
