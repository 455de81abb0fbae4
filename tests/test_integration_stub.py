"""The reference-side ctypes binding shown in INTEGRATION.md is executed
verbatim (extracted from the document) against a problem built with the
mirror modules, and must reproduce sumfac.assemble."""

import os
import re

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _stub_source():
    text = open(os.path.join(REPO, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# igasum/_b200\.py.*?)```", text, flags=re.S)
    assert m, "binding block missing from INTEGRATION.md"
    return m.group(1)


@pytest.mark.parametrize("d,p,K,kind", [(3, 4, 5, 3), (2, 3, 6, 2)])
def test_integration_stub_assembles_like_the_library(cuda, d, p, K, kind):
    from paper_1809_05471_b200 import sumfac, workloads

    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md", "exec"), ns)
    prob = workloads.make_problem(d, p, K, kind, seed=13)
    got = ns["assemble_values_b200"](prob)
    want = sumfac.assemble(prob).values_np()
    assert got.shape == want.shape
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
