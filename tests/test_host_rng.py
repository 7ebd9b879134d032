"""Host random source of generate_trace / the initial cache fill (inc/core.hpp:118-188): the
engine's bulk MT19937-64 must emit std::mt19937_64's words, and the threaded bulk normals must equal
sequential Box-Muller normal() calls bit for bit (tests/native/*.cpp, compiled here with g++)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2408_10284_b200", "csrc")


@pytest.mark.parametrize("name,extra", [("mt64_check", []),
                                        ("normals_check", [os.path.join(CSRC, "host", "policy.cpp"), "-lpthread"])])
def test_host_rng(name, extra, tmp_path):
    exe = tmp_path / name
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{CSRC}",
                    os.path.join(ROOT, "tests", "native", f"{name}.cpp"), *extra, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "OK", r.stdout + r.stderr
