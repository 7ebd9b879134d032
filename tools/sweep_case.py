"""Re-run one seed of tools/random_decode_sweep.py (debugging a mismatch): python tools/sweep_case.py SEED"""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("sweep", os.path.join(ROOT, "tools", "random_decode_sweep.py"))
m = importlib.util.module_from_spec(spec)
spec.loader.exec_module(m)
print(m.run(int(sys.argv[1])), flush=True)
