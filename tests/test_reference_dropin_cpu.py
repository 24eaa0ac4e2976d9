"""CPU checks of the reference-side B200 backend (integration/
hrt_b200_plugin.py) against the unmodified reference classes: the token
subclass constructs and behaves like CompletionToken (the reference
assigns ``status`` in ``__init__`` through ``__slots__``,
devices.py:206-214), the clock is a WallClock (comm.py:1035, 1045), and
with no GPU the backend refuses to start instead of falling back."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def plugin():
    if not os.path.isdir(os.path.join(REF, "hrt")):
        if not os.path.isdir("/root/reference/pkg"):
            pytest.skip("baseline/_ref (the reference install) is absent")
        subprocess.run(["sh", os.path.join(ROOT, "integration", "install_reference.sh")],
                       check=True, capture_output=True)
    for p in (REF, os.path.join(ROOT, "integration")):
        if p not in sys.path:
            sys.path.insert(0, p)
    import hrt_b200_plugin as P

    return P


def test_device_token_is_a_completion_token(plugin):
    from hrt.devices import CompletionToken, TokenKind, TokenStatus

    t = plugin.DeviceToken(7, TokenKind.KERNEL, 3)  # no event: behaves like the base class
    assert isinstance(t, CompletionToken)
    assert t.status is TokenStatus.PENDING and t.device_id == 3 and t.token_id == 7
    t._fire()  # the reference's own transition (devices.py:217-219)
    assert t.status is TokenStatus.COMPLETE
    t.status = TokenStatus.FAILED
    assert t.status is TokenStatus.FAILED


def test_device_clock_is_a_wall_clock(plugin):
    from hrt.devices import WallClock

    c = plugin.DeviceClock()
    assert isinstance(c, WallClock)
    assert c.advance_one() is None and c.pending_events == 0


def test_native_kernel_table_covers_the_reference_drivers(plugin):
    names = {"jacobi_update", "touch"} | {f"halo_{k}_{f}" for k in ("pack", "unpack")
                                          for f in range(6)}
    assert names <= set(plugin.NATIVE_KERNELS)


def test_no_gpu_means_loud_failure(plugin):
    from hrt.errors import HrtError

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(HrtError):
        plugin.lib()
