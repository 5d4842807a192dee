"""The C-ABI library loads and exports every symbol include/ellm.h declares (CPU-only)."""
import os
import re

from paper_2506_15155_b200 import ellm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ellm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ellm_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    names = declared()
    assert len(names) >= 30
    lib = ellm._lib
    for n in names:
        assert hasattr(lib, n), n
        assert n in ellm.EXPORTS, f"binding misses {n}"


def test_status_strings():
    assert ellm.status_string(0) == "ok"
    for rc in range(-1, -13, -1):
        assert ellm.status_string(rc) != "unknown status"


def test_no_device_pool_refuses_compute():
    p = ellm.Pool(ellm.DEVICE_NONE, 1, 4, 2, 64, 16, 8, 8, 2, 8, 4)
    assert p.reserve([0], [5]) == ellm.OK
    assert p.attention(0, [0], 0, 0, 1.0) == ellm.NO_DEVICE
    assert p.append(0, [0], [5], 0, 0) == ellm.NO_DEVICE
    assert p.base() == 0
    # knob validation happens before the device check
    assert p.set_swap_mode(4) == ellm.INVALID_ARG and p.set_swap_mode(-1) == ellm.INVALID_ARG
    assert p.set_swap_mode(2) == ellm.OK and p.set_swap_mode(3) == ellm.OK  # no side context without a device
    assert ellm.ellm_set_launch_overlap(p.handle, 2) == ellm.INVALID_ARG
    assert ellm.ellm_upload(p.handle, 1, 1, -1, None) == ellm.INVALID_ARG
    assert ellm.ellm_upload(p.handle, 1, 1, 8, None) == ellm.NO_DEVICE
    assert p.set_launch_overlap(True) == ellm.NO_DEVICE


def test_unsupported_shapes_rejected():
    import pytest
    for args in [(1, 4, 2, 96, 16), (1, 4, 2, 64, 24), (1, 32, 2, 64, 16), (1, 6, 3, 64, 16)]:
        with pytest.raises(ellm.EllmError) as e:
            ellm.Pool(ellm.DEVICE_NONE, *args, 8, 8, 2, 8, 0)
        assert e.value.rc == ellm.UNSUPPORTED
