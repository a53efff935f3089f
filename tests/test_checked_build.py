"""The kernels' own bounds checks (tools/gpu_checked.sh): compute-sanitizer is closed on the
GPU pool, so libprng_b200_checked.so (-DPRNG_CHECKED) checks every ring store and state
access of the seed / batch / epoch kernels against its launch's arguments and traps on a
violation.  Here: the negative control traps, and every kernel family's small case
(tools/sanitize_cases.py) runs clean and bit-exact against the oracle on the checked build.
The build's compiled-in traps are checked on CPU in tests/test_cabi_host.py."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ENV = dict(os.environ, PRNG_B200_CHECKED="1")

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SELFTEST = r"""
import ctypes, sys
import paper_1609_01257_b200 as P
L = P.lib()
assert P.LIB.endswith("libprng_b200_checked.so"), P.LIB
f = L.prng_checked_selftest
f.argtypes, f.restype = [ctypes.c_void_p, ctypes.POINTER(P.prng_err_t)], ctypes.c_int
h = P.prng_create(4096, 1)
err = P.prng_err_t()
rc = f(h, ctypes.byref(err))
print("selftest rc", rc, err.msg.decode(errors="replace"), flush=True)
sys.exit(0 if rc == P.PRNG_ECUDA else 1)
"""


def _run(args, timeout):
    return subprocess.run([sys.executable, *args], env=ENV, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module")
def checked_lib():
    r = _run(["-c", "from paper_1609_01257_b200 import _build; print(_build.build())"], 600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout.strip().splitlines()[-1]


def test_bounds_check_traps_on_an_overrun(checked_lib):
    """Negative control: a launch whose ring is 4 u64 short of the handle's count traps."""
    r = _run(["-c", SELFTEST], 300)
    assert r.returncode == 0, r.stdout + r.stderr[-3000:]
    assert "selftest rc -4" in r.stdout


def test_every_kernel_family_clean_on_the_checked_build(checked_lib):
    """tools/sanitize_cases.py (natural order with both barrier forms, ping-pong, time-parallel,
    epoch order, anti-absorption, star output, zero-copy, one-shot grids, fused and separate
    a1) on the checked build: no trap, and every case bit-exact against the oracle."""
    r = _run([os.path.join(ROOT, "tools", "sanitize_cases.py")], 900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "bounds violation" not in r.stdout + r.stderr
    assert r.stdout.count(" ok") >= 17 and "MISMATCH" not in r.stdout
