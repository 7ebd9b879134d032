"""CPU: both bench arms describe the run with the same `config` (the driver compares the reference
arm's line with ours), and the config holds only command-line / workload facts."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(argv):
    old = sys.argv
    sys.argv = ["bench.py"] + argv
    try:
        return bench.parse()
    finally:
        sys.argv = old


def test_static_config_is_argument_determined():
    for argv in ([], ["--batch", "16"], ["--store-format", "bf16"], ["--config", "mixtral-8x22b", "--layers", "16"],
                 ["--free-running"]):
        a = _args(argv)
        wl = bench.workload(a)
        c1, c2 = bench.static_config(a, wl, 1), bench.static_config(a, bench.workload(a), 1)
        assert c1 == c2
        assert c1["store_format"] == a.store_format and c1["batch"] == a.batch
        assert not {"tau", "capacities", "expert_store_per_rank"} & set(c1)
    a = _args([])
    assert a.store_format == "xbh"
    assert bench.static_config(a, bench.workload(a), 2)["parallelism"].startswith("ep2")
    assert bench.static_config(_args(["--replicas"]), bench.workload(a), 2)["parallelism"] == "replicas x2"
