"""The README's Python quick-start runs as written (GPU)."""

import os
import re

import pytest


@pytest.mark.gpu
def test_readme_quick_start_runs(cuda):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "README.md")
    code = re.search(r"```python\n(.*?)```", open(path).read(), re.S).group(1)
    exec(compile(code, "README.md", "exec"), {})
