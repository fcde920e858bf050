"""The reference's own test suite, run against the B200 path through the shim.

SURVEY.md 7.1 step 2: paper_1401_4068_b200.shim.install() rebinds the
reference's engine and estimator call sites (ente.ksg.batch_search,
ente.bench.batch_search, ente.inference.estimate_te_batch, ...) to this
package, then the reference's fast tests run unmodified:
/root/reference/pkg/tests/test_engine.py, test_ksg.py, test_inference.py,
test_bench.py (+ the remaining fast files, which exercise the reference's
host code in the same interpreter), and the quick acceptance criteria
(5: Gaussian analytic oracle, 6: engine O(n^2)-oracle equivalence).

The reference package and tests come from oracle/_ref/ente_ref.zip, staged
by __graft_entry__.build() from /root/reference (oracle/ref_stage.py); the
GPU box has no /root/reference.
"""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import ref_stage  # noqa: E402

PLUGIN = '''
import paper_1401_4068_b200.shim as shim
from paper_1401_4068_b200 import _native

import sys

def pytest_configure(config):
    _native.lib()          # the CUDA library must load: there is no fallback
    shim.install()
    import ente.ksg, ente.inference, ente.bench
    sys.stderr.write("B200 shim: ente.ksg.batch_search -> " +
                     ente.ksg.batch_search.__wrapped__.__module__ +
                     ", ente.inference.estimate_te_batch -> " +
                     ente.inference.estimate_te_batch.__wrapped__.__module__ + "\\n")
'''

FAST = ["test_engine.py", "test_ksg.py", "test_inference.py", "test_bench.py", "test_data.py",
        "test_embedding.py", "test_io_cli.py", "test_simulators.py"]


def _run(tmp_path, targets, timeout):
    root = ref_stage.extract(str(tmp_path / "ref"))
    if root is None:
        pytest.skip("reference not staged (oracle/_ref/ente_ref.zip: run __graft_entry__.build() "
                    "where /root/reference exists)")
    (tmp_path / "ente_b200_shim_plugin.py").write_text(PLUGIN)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(tmp_path), os.path.join(root, "src"), ROOT])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba_cache")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ente_b200_shim_plugin",
           "-p", "no:cacheprovider", "-rs"] + [os.path.join(root, "tests", t) for t in targets]
    r = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True,
                       timeout=timeout)
    out = r.stdout + r.stderr
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log") if
              os.path.isdir(os.path.join(ROOT, "gpurun_out")) else os.devnull, "a") as f:
        f.write(" ".join(targets) + "\n" + out + "\n")
    passed = int(m.group(1)) if (m := re.search(r"(\d+) passed", out)) else 0
    return r.returncode, passed, out


@pytest.mark.gpu
def test_reference_fast_suite_through_shim(tmp_path):
    rc, passed, out = _run(tmp_path, FAST, timeout=1800)
    assert "B200 shim: ente.ksg.batch_search -> paper_1401_4068_b200.engine" in out, out[-3000:]
    assert rc == 0, out[-6000:]
    assert passed >= 93, out[-3000:]


@pytest.mark.gpu
def test_reference_acceptance_5_and_6_through_shim(tmp_path):
    rc, passed, out = _run(tmp_path, ["test_acceptance.py::test_criterion_5_gaussian_analytic_oracle",
                                      "test_acceptance.py::test_criterion_6_engine_oracle_equivalence"],
                           timeout=1800)
    assert rc == 0, out[-6000:]
    assert passed == 2, out[-3000:]
