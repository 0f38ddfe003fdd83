"""bench.py plumbing that runs without a GPU: the reference arm is the
reference's own CPU path and never loads the product library; `--gpus N`
re-executes itself under torch.distributed.run with one rank per GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

import oracle as O  # noqa: E402

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

PROBE = r"""
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", sys.argv[1], "--steps", "2"]
sys.path.insert(0, {root!r})
import bench
rc = bench.main()
maps = open("/proc/self/maps").read()
libs = sorted(set(l.split()[-1] for l in maps.splitlines() if l.endswith(".so")
                   and {root!r} in l))
print(json.dumps({{"rc": rc, "libs": libs,
                   "product_imported": "paper_2409_02208_b200" in sys.modules}}))
"""


def _run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    if env:
        e.update(env)
    return subprocess.run([sys.executable] + args, capture_output=True, text=True, cwd=ROOT,
                          env=e, timeout=timeout)


@needs_ref
@pytest.mark.parametrize("config", ["cfg0", "cfg1"])
def test_reference_arm_loads_only_oracle_libraries(config):
    r = _run(["-c", PROBE.format(root=ROOT), config])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"] == config
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert probe["rc"] == 0 and not probe["product_imported"]
    assert probe["libs"], "the reference library was not loaded"
    for lib in probe["libs"]:
        assert "/oracle/" in lib, lib


@needs_ref
def test_gpus_flag_relaunches_one_rank_per_gpu():
    # the reference arm under the launcher: rank 0 prints, rank 1 exits 0
    r = _run(["bench.py", "--impl", "reference", "--gpus", "2", "--config", "cfg0",
              "--steps", "1"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def test_world_size_must_match_gpus_flag():
    r = _run(["bench.py", "--impl", "reference", "--gpus", "4", "--config", "cfg0"],
             env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_parity_gate_modes():
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    a = np.arange(12, dtype=np.float32).reshape(3, 4)
    assert bench.parity(a, a.copy(), exact=True)["ok"]
    b = a.copy()
    b[1, 2] = np.nextafter(b[1, 2], np.float32(100))
    assert not bench.parity(b, a, exact=True)["ok"]
    assert bench.parity(b, a, exact=False)["ok"]          # 1 ulp: normwise ok
    c = a.copy()
    c[0, 0] += 1e-3
    assert not bench.parity(c, a, exact=False)["ok"]       # 1e-3/11 > 1e-5
