"""Both forms of kernel (2) against the oracle: the library picks the warp-MMA
fold for flushes / compressions (and commits whose slots all hold records)
and the tcgen05 fold for the other commits (csrc/fold.cu).
LABUF_FOLD=tc|wm forces one form for every fold kind; it is read once per
process, so each form runs the fold-heavy parity files in a subprocess."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = ["tests/test_gpu_parity.py", "tests/test_gpu_paged.py", "tests/test_gpu_multiround.py",
         "tests/test_gpu_parity_fp32_edges.py"]


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["tc", "wm"])
def test_fold_form_forced(form):
    env = dict(os.environ, LABUF_FOLD=form)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", *FILES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, f"LABUF_FOLD={form}:\n{r.stdout[-3000:]}\n{r.stderr[-2000:]}"
