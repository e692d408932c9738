"""Run the reference's OWN test suite against this package (API parity).

The reference tests (/root/reference/pkg/tests, 125 tests incl. hypothesis
property suites at 1,000 cases and acceptance criteria 1-9) are copied to a
temp dir next to a conftest that aliases `gpumux.device`, `gpumux.kernels`,
`gpumux.coalesce` and `gpumux.scheduler` to this package's modules before
`gpumux` is imported. The reference's engine/cli/rng/tuning modules then run
on top of the native decision core, so every engine-level test (trace
determinism, acceptance criteria 1/2/6/8, the 1,000-case run invariants)
exercises the product. Build container only (needs the reference tree).
"""

import os
import shutil
import subprocess
import sys

import pytest

from .conftest import REF_SRC, REPO, reference_available

ALIAS_CONFTEST = '''
import sys
sys.path.insert(0, {repo!r})
sys.path.insert(0, {ref!r})
import paper_1901_10008_b200.device as _d
import paper_1901_10008_b200.kernels as _k
import paper_1901_10008_b200.coalesce as _c
import paper_1901_10008_b200.scheduler as _s
sys.modules["gpumux.device"] = _d
sys.modules["gpumux.kernels"] = _k
sys.modules["gpumux.coalesce"] = _c
sys.modules["gpumux.scheduler"] = _s
import gpumux
for _n, _m in (("device", _d), ("kernels", _k), ("coalesce", _c), ("scheduler", _s)):
    setattr(gpumux, _n, _m)
import gpumux.engine
assert gpumux.engine.Scheduler is _s.Scheduler
'''


@pytest.mark.reference
@pytest.mark.skipif(not reference_available(), reason="reference tree not present")
def test_reference_suite_passes_on_product(tmp_path):
    dst = tmp_path / "reftests"
    shutil.copytree(os.path.join(os.path.dirname(REF_SRC), "tests"), dst)
    (dst / "conftest.py").write_text(ALIAS_CONFTEST.format(repo=REPO, ref=REF_SRC))
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REPO, REF_SRC]))
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           "-x", str(dst)], capture_output=True, text=True, env=env,
                          cwd=str(tmp_path), timeout=1800)
    tail = "\n".join(proc.stdout.strip().splitlines()[-15:])
    assert proc.returncode == 0, tail
    assert "125 passed" in tail and "failed" not in tail, tail
