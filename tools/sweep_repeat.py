"""Run one seed of tools/random_decode_sweep.py REPS times in one process (race hunting)."""
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("sweep", os.path.join(ROOT, "tools", "random_decode_sweep.py"))
m = importlib.util.module_from_spec(spec)
spec.loader.exec_module(m)
seed, reps = int(sys.argv[1]), int(sys.argv[2])
bad = 0
for i in range(reps):
    try:
        ok, why = m.run(seed)
    except Exception as e:  # noqa: BLE001
        ok, why = False, repr(e)[:200]
    if not ok:
        bad += 1
        print("FAIL", i, why, flush=True)
        if "illegal" in why:
            break
print(f"seed {seed}: {reps - bad} / {reps} ok", flush=True)
