"""The reference's own acceptance gate (tests/acceptance.cpp:122-584), compiled
unchanged against tucker_gpu (paper_2308_16395_b200/shim): the reference's
streaming API served by the B200 path through include/tsg.h. Criteria 1-3
and 6-8 drive stream_init / stream_update / full_model on the GPU;
criterion 4 exercises add_row / isvd_init, which stay the reference
library's own; criterion 5 needs the reference CLI (absent: CLI11 is not
vendored), so it fails on the CPU build as well."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GATE = os.path.join(ROOT, "paper_2308_16395_b200", "shim", "_build", "acceptance_gpu")


def test_reference_acceptance_gate_through_gpu_shim():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(GATE):
        pytest.skip("shim/_build/acceptance_gpu not built (needs the reference sources)")
    p = subprocess.run([GATE], capture_output=True, text=True, timeout=900)
    print(p.stdout[-4000:])
    assert p.returncode >= 0, f"acceptance_gpu died with signal {-p.returncode}"
    res = dict((int(i), s) for s, i in re.findall(r"\[(PASS|FAIL)\] (\d)\.", p.stdout))
    assert len(res) == 8, p.stdout[-2000:]
    # 5: the CLI binary is not buildable here (TUCKER_CLI unset)
    failed = sorted(i for i, s in res.items() if s == "FAIL" and i != 5)
    assert not failed, f"criteria {failed} failed:\n{p.stdout[-3000:]}"
