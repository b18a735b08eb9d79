"""CPU-only checks of the C ABI library: it loads without a GPU, exports every
symbol include/dmha.h declares, reports state errors instead of crashing, and
its host index math (hot-path step a1) is right."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2302_06218_b200 import dmha

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).parent / "golden" / "shard_layouts.txt"


def header_symbols():
    text = (ROOT / "include" / "dmha.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(dmha_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = dmha.lib()
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert set(syms) == set(dmha.EXPORTED_SYMBOLS)


def test_calls_before_init_return_state_error():
    with pytest.raises(dmha.DmhaError) as e:
        dmha.workspace_bytes(1024, 64, 2)
    assert e.value.code == dmha.ERR_STATE
    with pytest.raises(dmha.DmhaError) as e:
        dmha.synchronize()
    assert e.value.code == dmha.ERR_STATE
    rc = dmha.lib().dmha_forward(None, None, None, None, None, 128, 64, 1, 0)
    assert rc == dmha.ERR_STATE
    assert b"not initialised" in dmha.lib().dmha_last_error()


def test_init_argument_validation_without_gpu():
    lib = dmha.lib()
    assert lib.dmha_init(0, 0, None, 0, 0, 0, None) == dmha.ERR_INVALID
    assert lib.dmha_init(2, 0, None, 0, 0, 0, None) == dmha.ERR_INVALID  # needs unique id
    assert lib.dmha_init(1, 0, None, 0, 7, 0, None) == dmha.ERR_INVALID  # bad dtype
    assert lib.dmha_init(1, 0, None, 0, 0, 9, None) == dmha.ERR_INVALID  # bad layout


def _golden_layouts():
    for line in GOLDEN.read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            name, L, P, lay, rows = [s.strip() for s in line.split("|")]
            yield name, int(L), int(P), lay, [[int(x) for x in r.split()] for r in rows.split(";")]


@pytest.mark.parametrize("case", list(_golden_layouts()), ids=lambda c: c[0])
def test_shard_layout_golden(case):
    name, L, P, lay, expect = case
    for r in range(P):
        got_c = [dmha.local_to_global(L, P, r, lay, i) for i in range(L // P)]
        assert got_c == expect[r]
        assert dmha.global_rows(L, P, r, lay).tolist() == expect[r]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("layout", ["contiguous", "zigzag"])
def test_layout_is_a_partition_and_increasing(P, layout):
    L = 2 * P * 37
    allrows = []
    for r in range(P):
        g = dmha.global_rows(L, P, r, layout)
        assert np.all(np.diff(g) > 0)            # increasing local->global map
        for i in (0, len(g) // 2, len(g) - 1):
            assert dmha.local_to_global(L, P, r, layout, i) == g[i]
        allrows.append(g)
    allrows = np.concatenate(allrows)
    assert np.array_equal(np.sort(allrows), np.arange(L))


def test_zigzag_balances_causal_work_exactly():
    """Causal pair counts per rank: zigzag equal across ranks, contiguous not
    (max/mean 1.874 at P=8)."""
    L, P = 1024, 8
    for layout, balanced in (("zigzag", True), ("contiguous", False)):
        work = [int((dmha.global_rows(L, P, r, layout) + 1).sum()) for r in range(P)]
        assert (max(work) == min(work)) == balanced


def test_shard_unshard_roundtrip():
    x = np.arange(48 * 3).reshape(48, 3)
    for layout in ("contiguous", "zigzag"):
        parts = [dmha.shard(x, 4, r, layout) for r in range(4)]
        np.testing.assert_array_equal(dmha.unshard(parts, 48, layout), x)


def test_uneven_contiguous_shards_follow_spec_example():
    """SPEC S:445's equal-as-possible partition: L = 10 over 4 workers is
    {3, 3, 2, 2} rows, in order (rank r starts at r*(L/P) + min(r, L % P))."""
    assert [dmha.shard_rows(10, 4, r, "contiguous") for r in range(4)] == [3, 3, 2, 2]
    rows = [list(dmha.global_rows(10, 4, r, "contiguous")) for r in range(4)]
    assert rows == [[0, 1, 2], [3, 4, 5], [6, 7], [8, 9]]
    assert [dmha.local_to_global(10, 4, 2, "contiguous", i) for i in range(2)] == [6, 7]
    with pytest.raises(dmha.DmhaError):
        dmha.local_to_global(10, 4, 2, "contiguous", 2)   # rank 2 owns 2 rows
    # every L and P: the shards partition [0, L) in order, sizes differ by <= 1
    for L in range(1, 40):
        for P in range(1, 9):
            g = np.concatenate([dmha.global_rows(L, P, r, "contiguous") for r in range(P)])
            assert np.array_equal(g, np.arange(L))
            sz = [dmha.shard_rows(L, P, r, "contiguous") for r in range(P)]
            assert max(sz) - min(sz) <= 1


def test_bad_layout_args():
    with pytest.raises(dmha.DmhaError):
        dmha.local_to_global(12, 4, 0, "zigzag", 0)       # 12 % 8 != 0
    with pytest.raises(dmha.DmhaError):
        dmha.local_to_global(16, 4, 4, "zigzag", 0)       # rank out of range


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No fallback: without libdmha.so every call raises DmhaError (the
    product never routes through the oracle or a CPU path)."""
    from paper_2302_06218_b200 import dmha
    monkeypatch.setattr(dmha, "_lib", None)
    monkeypatch.setattr(dmha, "_LIB_PATH", tmp_path / "libdmha.so")
    with pytest.raises(dmha.DmhaError):
        dmha.lib()
    with pytest.raises(dmha.DmhaError):
        dmha.workspace_bytes(1024, 64, 2)


def test_product_does_not_import_the_oracle():
    """The product package (binding and CUDA sources) never imports, links or
    includes anything under oracle/ (comments may mention it)."""
    import pathlib
    import re
    root = pathlib.Path(__file__).resolve().parent.parent / "paper_2302_06218_b200"
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle|#\s*include\s*[<\"].*oracle)", re.M)
    files = list(root.glob("*.py")) + [f for f in (root / "csrc").glob("*") if f.is_file()]
    assert files
    for f in files:
        assert not pat.search(f.read_text(errors="ignore")), f
    assert "oracle" not in (root / "build.py").read_text()
