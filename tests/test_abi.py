"""The C-ABI library loads and exports every symbol include/*.h declares (CPU).

No compute call is made here (there is no GPU in the build container); only
the host-side argument checks that return before any CUDA call are exercised.
"""
import ctypes
import glob
import os
import re
import subprocess

import pytest

from paper_2002_05200_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


def header_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(\w+)\s*\([^;{]*\)\s*;", text):
            if m.group(1) not in ("if", "sizeof"):
                names.add(m.group(1))
    return names


def test_header_declares_the_binding_exports():
    assert header_functions() == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in header_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_side_checks_without_gpu(lib):
    assert lib.logan_abi_version() == 3
    # window widths by level (diagnostics; results never depend on them)
    assert lib.logan_level_width(1, 20, 2500, 0) == 32 and lib.logan_level_width(1, 20, 10000, 0) == 32
    assert lib.logan_level_width(1, 20, 7700, 0) == 32 and lib.logan_level_width(1, 18, 7700, 0) == 32
    assert lib.logan_level_width(1, 10, 2500, 0) == 24 and lib.logan_level_width(1, 20, 2500, 24) == 24
    assert [lib.logan_level_width(1, x, 2500, 0) for x in (0, 5, 6, 10, 11, 12, 16)] == [16, 16, 24, 24, 32, 32, 32]
    assert lib.logan_level_width(1, 10, 10000, 0) == 24 and lib.logan_level_width(1, 20, 2500, 16) == 16
    assert [lib.logan_level_width(lv, 50, 2500, 0) for lv in range(2, 6)] == [64, 128, 256, 512]
    assert [lib.logan_level_width(6, x, 2500, 0) for x in (50, 500, 600, 700, 1000)] == [1024, 640, 768, 896, 1024]
    assert lib.logan_level_width(7, 5000, 2500, 0) == 0 and lib.logan_level_width(0, 20, 2500, 0) == 0
    assert lib.logan_strerror(1) == b"invalid argument"
    assert lib.logan_workspace_bytes(-1, 0) == 0
    small, big = lib.logan_workspace_bytes(10, 100), lib.logan_workspace_bytes(1000, 100)
    assert 0 < small < big
    assert lib.logan_workspace_bytes(10, 1000) > small  # wide-level scratch grows with length
    sc_bad = _lib.Scoring(1, 1, -1, 10)  # mismatch must be < 0
    st = lib.logan_xdrop_batch(None, 1, 0, None, None, None, None, None, None, 5, 0, 17, sc_bad,
                               None, None, None, None, None, 0, None)
    assert st == _lib.LOGAN_EINVAL
    sc = _lib.Scoring(1, -1, -1, 10)
    st = lib.logan_xdrop_batch(None, 7, 0, None, None, None, None, None, None, 5, 0, 17, sc,
                               None, None, None, None, None, 0, None)
    assert st == _lib.LOGAN_EINVAL  # unknown format
    st = lib.logan_xdrop_batch(None, 1, 0, None, None, None, None, None, None, 0, 0, 17, sc,
                               None, None, None, None, None, 0, None)
    assert st == _lib.LOGAN_OK  # n_pairs = 0: no-op, nothing launched
    st = lib.logan_xdrop_batch(None, 1, 0, None, None, None, None, None, None, 3, 0, 17, sc,
                               None, None, None, None, None, 0, None)
    assert st == _lib.LOGAN_EINVAL  # NULL device pointers
    # substitution matrices: u8 pool only, 1 <= alphabet <= 32 (checked before any launch)
    opt = _lib.Options()
    opt.subst = 0x1000
    opt.alphabet = 20
    st = lib.logan_xdrop_batch(None, 1, 0, None, None, None, None, None, None, 3, 0, 17, sc,
                               ctypes.byref(opt), None, None, None, None, 0, None)
    assert st == _lib.LOGAN_EINVAL  # 2-bit pool with a matrix
    opt.alphabet = 33
    st = lib.logan_xdrop_batch(None, 0, 0, None, None, None, None, None, None, 3, 0, 17, sc,
                               ctypes.byref(opt), None, None, None, None, 0, None)
    assert st == _lib.LOGAN_EINVAL  # alphabet too large
    assert ctypes.sizeof(_lib.Options) == 64  # layout of logan_options_t


def test_workspace_and_bounds_checked_before_launch(lib):
    """ABI v2: the workspace must hold logan_workspace_bytes(n_pairs, max_ext_len)
    (else LOGAN_ENOSPC, synchronously, nothing launched); X and Z up to 2^28 are
    accepted, beyond is LOGAN_EINVAL; max_ext_len must be in [0, 2^30). The fake
    device pointers below are never dereferenced: every check returns first."""
    sc = _lib.Scoring(1, -1, -1, 20)
    fake = 0x100000  # 256-byte aligned, non-NULL
    args = lambda n, ext, sc_, ws_bytes, opt=None: (fake, 1, 1000, fake, fake, fake, fake, fake, fake, n, ext, 17,
                                                    sc_, opt, fake, None, None, fake, ws_bytes, None)
    need = lib.logan_workspace_bytes(100, 5000)
    assert lib.logan_xdrop_batch(*args(100, 5000, sc, need - 1)) == _lib.LOGAN_ENOSPC
    # a workspace sized for shorter extensions than the declared bound is refused
    assert lib.logan_xdrop_batch(*args(100, 5000, sc, lib.logan_workspace_bytes(100, 100))) == _lib.LOGAN_ENOSPC
    assert lib.logan_xdrop_batch(*args(100, -1, sc, need)) == _lib.LOGAN_EINVAL
    assert lib.logan_xdrop_batch(*args(100, 1 << 30, sc, need)) == _lib.LOGAN_EINVAL
    assert lib.logan_xdrop_batch(*args(100, 5000, _lib.Scoring(1, -1, -1, (1 << 28) + 1), need)) == _lib.LOGAN_EINVAL
    assert lib.logan_xdrop_batch(*args(100, 5000, _lib.Scoring(1, -1, -1, -1), need)) == _lib.LOGAN_EINVAL
    opt = _lib.Options()
    opt.flags = 4
    opt.zdrop = (1 << 28) + 1
    assert lib.logan_xdrop_batch(*args(100, 5000, sc, need, ctypes.byref(opt))) == _lib.LOGAN_EINVAL
    # the host entry point: an arena smaller than the copies it needs
    st = lib.logan_xdrop_batch_host(fake, 1, 1000, fake, fake, fake, fake, fake, fake, 0, 17, sc, None, fake,
                                    None, fake, 0, None)
    assert st == _lib.LOGAN_OK  # n_pairs = 0: no-op


def test_product_path_does_not_import_oracle():
    """The product package never references oracle/ (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2002_05200_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if path.endswith((".py", ".cu", ".cuh", ".h")):
            text = open(path).read()
            assert "import oracle" not in text and "from oracle" not in text, path
            assert "xdrop_oracle" not in text, path


def test_pack_2bit_host_checks_without_gpu(lib):
    # size: ceil(pool_len / 16) packed words plus 16 bytes of zero padding
    assert [lib.logan_pack_2bit_bytes(n) for n in (0, 1, 16, 17, 1000)] == [16, 20, 20, 24, 268]
    assert lib.logan_pack_2bit_bytes(-1) == 0
    fake = 1 << 20  # never dereferenced: every check below returns before any CUDA call
    d = (fake, fake, fake, fake)  # read descriptors

    def pk(u8, n, desc, npairs, out, nb, other):
        return lib.logan_pack_2bit(u8, n, *desc, npairs, out, nb, other, None)
    assert pk(fake, -1, d, 1, fake, 64, fake) == _lib.LOGAN_EINVAL
    assert pk(fake, 100, d, -1, fake, 64, fake) == _lib.LOGAN_EINVAL
    assert pk(fake, 100, d, 1, fake, 64, None) == _lib.LOGAN_EINVAL
    assert pk(fake, 100, d, 1, fake, 64, fake + 4) == _lib.LOGAN_EINVAL  # n_other misaligned
    assert pk(None, 100, d, 1, fake, 64, fake) == _lib.LOGAN_EINVAL
    assert pk(fake + 2, 100, d, 1, fake, 64, fake) == _lib.LOGAN_EINVAL
    assert pk(fake, 100, (fake, None, fake, fake), 1, fake, 64, fake) == _lib.LOGAN_EINVAL
    assert pk(fake, 100, d, 1, fake, 39, fake) == _lib.LOGAN_ENOSPC
    # the host arena of a u8 pool includes the packed copy (the synchronous entry packs)
    a8 = lib.logan_host_arena_bytes(100, 4000, _lib.LOGAN_SEQ_U8, 100)
    a2 = lib.logan_host_arena_bytes(100, 4000, _lib.LOGAN_SEQ_2BIT, 100)
    assert a8 >= a2 + 4000 - 1000 + lib.logan_pack_2bit_bytes(4000)
