"""CPU: the parts of bench.py's contract that need no GPU -- the reference arm
(`--impl reference`) end to end on the small config, and the workload
description both arms print."""
import json
import os
import subprocess
import sys
import types

from conftest import ROOT


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--gpus", "1", "--steps", "6", "--warmup", "3"],
                         capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr[-400:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "sweeps/s" and d["higher_is_better"] is True
    assert d["steps"] == 6 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and abs(d["ms_per_step"] * d["value"] - 1e3) < 1e-6
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"] == {"value": d["value"], "unit": "sweeps/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["vs_baseline"] is None and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("c1:")


def test_both_arms_describe_the_same_config():
    sys.path.insert(0, ROOT)
    import bench
    for name in ("c1", "c2", "c4", "c5"):
        args = types.SimpleNamespace(config=name, gpus=1)
        c = bench.CONFIGS[name]
        a = bench.bench_config(args, c, 1)
        assert a == bench.bench_config(args, c, max(1, args.gpus))
        assert a["dims"] == list(c["dims"]) and a["rank"] == c["rank"]
        big = 8 * int(__import__("numpy").prod(c["dims"])) > 126e6
        assert ("streams X from HBM" in a["l2"]) == big  # truthful about L2 residency
    # the sharded description names the world size
    assert "x4" in bench.bench_config(types.SimpleNamespace(config="c5", gpus=4),
                                      bench.CONFIGS["c5"], 4)["parallelism"]
