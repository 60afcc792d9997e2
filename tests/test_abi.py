"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/ara.h declares, and its host-only helpers follow the DESIGN.md readings."""
import math
import os
import re
import subprocess
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ara.h")
LIB = os.path.join(ROOT, "paper_1606_04473_b200", "libara.so")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:ara_status|void|uint64_t|const char\*|char\*)\s*\**\s*(ara_\w+)\s*\(",
                                 src, flags=re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libara.so not built"
    syms = declared_symbols()
    assert len(syms) >= 13, syms
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    from paper_1606_04473_b200 import ara
    assert set(syms) == set(ara.EXPORTED)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_partition_matches_reading_a17():
    from paper_1606_04473_b200 import ara
    for T in (0, 1, 7, 1000, 1_000_000, 10_000_001):
        for N in (1, 2, 3, 4, 8, 16):
            got = [ara.ara_partition(T, N, r) for r in range(N)]
            sizes = [c for _, c in got]
            assert sum(sizes) == T and max(sizes) - min(sizes) <= 1
            assert all(got[r][0] == sum(sizes[:r]) for r in range(N))
            assert sizes == sorted(sizes, reverse=True)
    with pytest.raises(ara.AraError):
        ara.ara_partition(10, 2, 2)


def test_return_period_rank_is_exact_ceiling():
    """A10: k = ceil(T/R) computed exactly (checked with rationals)."""
    from paper_1606_04473_b200 import ara
    rng = np.random.default_rng(2)
    for _ in range(3000):
        T = int(rng.integers(1, 10_000_000))
        R = float(rng.integers(1, T + 1)) if rng.random() < 0.5 else float(rng.uniform(1, T))
        assert ara.ara_return_period_rank(T, R) == math.ceil(Fraction(T) / Fraction(R))
    for bad in (0.0, 0.999, 11.0, float("nan"), float("inf")):
        with pytest.raises(ara.AraError) as ei:
            ara.ara_return_period_rank(10, bad)
        assert ei.value.status == ara.ARA_ERR_DOMAIN


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1606_04473_b200 import ara
    with pytest.raises(ara.AraError) as ei:
        ara.Context(1000)
    assert ei.value.status == ara.ARA_ERR_CUDA


def test_invalid_config_rejected_before_touching_the_gpu():
    from paper_1606_04473_b200 import ara
    for kw in ({"world": 2}, {"rank": 1}, {"precision": 7}):
        with pytest.raises(ara.AraError) as ei:
            ara.ara_create(1000, **kw)
        assert ei.value.status == ara.ARA_ERR_INVALID_ARG
    with pytest.raises(ara.AraError):
        ara.ara_create(0)


def test_product_path_never_touches_the_oracle():
    """The oracle is test infrastructure: no product source may import, link or
    call it, and no CPU fallback exists."""
    pkg = os.path.join(ROOT, "paper_1606_04473_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "oracle.h", "oracle_"):
                    assert bad not in txt, (f, bad)
    out = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "oracle" not in out


def test_pack_ids_matches_bit_layout():
    """F3 packed transfer format: id i at bit offset i*bits, little-endian words."""
    from paper_1606_04473_b200 import ara
    rng = np.random.default_rng(5)
    for bits in (1, 7, 21, 31, 32):
        for n in (0, 1, 31, 32, 33, 1000, (1 << 20) + 77):
            ids = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(np.uint32)
            packed = ara.ara_pack_ids(ids, bits)
            assert len(packed) == (n * bits + 31) // 32 + 1
            # decode with python big ints on a sample (exhaustive for small n)
            as_int = int.from_bytes(packed.astype("<u4").tobytes(), "little")
            idx = range(n) if n <= 2000 else rng.integers(0, n, 2000)
            for i in idx:
                assert (as_int >> (int(i) * bits)) & ((1 << bits) - 1) == ids[i]
    with pytest.raises(ara.AraError):
        ara.ara_pack_ids(np.array([1 << 21], np.uint32), 21)


def test_binding_structs_match_the_c_header(tmp_path):
    """The ctypes mirrors of the ABI structs have the C header's size and field
    offsets (a mismatch would silently corrupt arguments or stats)."""
    import ctypes
    import subprocess
    from paper_1606_04473_b200 import ara
    structs = {"ara_config": ara.ara_config, "ara_elt_terms": ara.ara_elt_terms, "ara_layer": ara.ara_layer,
               "ara_layer_list": ara.ara_layer_list, "ara_run_stats": ara.ara_run_stats}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "ara.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n"):
        if line:
            n, f, v = line.split()
            got[(n, f)] = int(v)
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[(name, f)] == getattr(cls, f).offset, (name, f)
