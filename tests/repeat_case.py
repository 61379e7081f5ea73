"""Run one replay-step parity case repeatedly (flake hunting):
    python tests/repeat_case.py <case> [reps]   (test infrastructure: uses the oracle)"""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.pyoracle import Oracle  # noqa: E402
from tests.harness import StepConfig, run_step_parity  # noqa: E402
from tests.test_gpu_parity import STEP_CASES  # noqa: E402

case = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ora = Oracle()
if STEP_CASES[case].get("early_gather"):
    os.environ["RB_EARLY_GATHER"] = "1"
bad = 0
for r in range(reps):
    try:
        run_step_parity(StepConfig(**STEP_CASES[case]), steps=12, ora=ora)
    except AssertionError:
        bad += 1
        if bad <= 3:
            traceback.print_exc(limit=1)
print(f"{case}: {bad}/{reps} failed")
