"""The reference's OWN test-suite (pkg/tests, copied into oracle/_ref by
oracle/make_ref.py) run against the reference package with the B200 drop-in
installed (tests/neo_dropin_plugin.py): every forward_pooled / fused_forward /
backward_sort_aggregate / optimizer / fused_backward_update / bucketize /
permute / redistribute / train_step_* / simulate_trace call the suite makes
goes through libneob200 on the GPU, in f64 (bit-exact mode).  SURVEY.md 4:
test_embedding.py, test_comms.py (incl. the sharded-step equivalence at
:318-419), test_acceptance.py criteria 5 (:202-247) and 6 (:250-285) and
the rest of the suite."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
MODULES = ["test_embedding.py", "test_comms.py", "test_acceptance.py", "test_cache.py", "test_core.py",
           "test_cli.py", "test_planner.py", "test_perf.py"]


@pytest.mark.parametrize("module", MODULES)
def test_reference_suite_through_dropin(module):
    if not (REF / "tests" / module).exists():
        pytest.fail("oracle/_ref is missing: run __graft_entry__.build() (oracle/make_ref.py) where "
                    "/root/reference exists")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ROOT), str(REF), env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "neo_dropin_plugin", "-p", "no:cacheprovider",
                        "--rootdir", str(REF), "-c", os.devnull, str(REF / "tests" / module)],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    tail = "\n".join(out.strip().splitlines()[-25:])
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) > 0, tail
    assert "dropin: CUDA device used" in out, tail
    print(f"{module}: {m.group(0)} through the drop-in")
