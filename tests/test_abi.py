"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/fdwave_cuda.h declares, and the host-only helpers (slab
split, owner lookup, descriptor defaults, create-time validation) behave."""
import ctypes as C
import os
import re

import pytest

from paper_2201_05278_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdwave_cuda.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdw_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_solver_surface():
    names = declared()
    for n in ["fdw_create", "fdw_set_medium", "fdw_set_sources", "fdw_set_receivers", "fdw_advance",
              "fdw_refresh_boundary", "fdw_record", "fdw_max_abs", "fdw_get_levels", "fdw_set_levels",
              "fdw_download_seismogram", "fdw_destroy"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared()) == set(_lib.EXPORTED)


def test_desc_layout_matches_c():
    # the C side memsets sizeof(fdw_desc); a ctypes mismatch would corrupt fields
    d = _lib.fdw_desc()
    _lib.lib().fdw_desc_init(C.byref(d))
    assert d.abi_version == _lib.FDW_ABI_VERSION
    assert d.check_interval == 100 and d.world == 1 and d.dtype_bytes == 4
    assert C.sizeof(_lib.fdw_desc) == 320


@pytest.mark.parametrize("n,world", [(217, 1), (217, 2), (217, 8), (1600, 8), (19, 3)])
def test_slab_range_partitions_planes(n, world):
    L = _lib.lib()
    prev_end = 0
    sizes = []
    for r in range(world):
        b, e = C.c_uint64(), C.c_uint64()
        assert L.fdw_slab_range(n, world, r, C.byref(b), C.byref(e)) == 0
        assert b.value == prev_end and e.value > b.value
        sizes.append(e.value - b.value)
        prev_end = e.value
    assert prev_end == n and max(sizes) - min(sizes) <= 1


def test_owner_of_matches_slab_range():
    L = _lib.lib()
    ext = (C.c_uint64 * 3)(40, 9, 7)
    h, world = 4, 3
    P1, P2 = 9 + 8, 7 + 8
    for z in range(-h, 40 + h):
        flat = ((z + h) * P1 + 5) * P2 + 6
        owner = L.fdw_owner_of(flat, ext, h, world)
        if z < 0 or z >= 40:
            assert owner == -1
        else:
            b, e = C.c_uint64(), C.c_uint64()
            L.fdw_slab_range(40, world, owner, C.byref(b), C.byref(e))
            assert b.value <= z < e.value


def test_create_rejects_bad_descriptors_without_touching_the_gpu():
    L = _lib.lib()
    for field, value in (("ndim", 4), ("space_order", 7), ("dtype_bytes", 2), ("abi_version", 99)):
        d = _lib.fdw_desc()
        L.fdw_desc_init(C.byref(d))
        d.extended[0] = d.extended[1] = d.extended[2] = 32
        setattr(d, field, value)
        h = C.c_void_p()
        assert L.fdw_create(C.byref(d), C.byref(h)) == _lib.FDW_EINVAL
        assert L.fdw_last_error(None)
    d = _lib.fdw_desc()
    L.fdw_desc_init(C.byref(d))
    d.extended[0], d.extended[1], d.extended[2] = 9, 32, 32  # 9 < 2*4+2
    assert L.fdw_create(C.byref(d), C.byref(C.c_void_p())) == _lib.FDW_EINVAL
    assert b"2*halo+2" in L.fdw_last_error(None)


def test_library_needs_no_nccl():
    """The halo exchange is peer memory, not NCCL: the library links no NCCL."""
    import subprocess
    r = subprocess.run(["readelf", "-d", _lib.LIB_PATH], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    assert "nccl" not in r.stdout.lower(), r.stdout


def test_library_then_torch_import_order():
    """Loading the library before torch must not disturb torch's own NCCL."""
    import subprocess
    import sys
    code = ("from paper_2201_05278_b200 import _lib; _lib.lib(); import torch; "
            "import torch.distributed as d; print(d.is_nccl_available())")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
