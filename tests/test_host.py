"""CPU: the C ABI library loads and exports every declared symbol, host-side
logic (validation, schedules, metrics, containers, file formats, partition
math) matches the reference's, and operators fail loudly without a GPU."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    text = (ROOT / "include" / "halfgnn.h").read_text()
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2411_01109_b200 import _native

    lib = _native.lib()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_native.SIGNATURES), "ctypes table out of sync with header"
    assert lib.hg_abi_version() == 6


def test_library_workspace_queries_without_gpu():
    from paper_2411_01109_b200 import _native

    # (the CUB-backed sizing queries need a device; these are pure arithmetic)
    assert _native.size_query("hg_spmm_workspace", 100, 64, 10, 1, 1, 0) >= 100 * 64 * 2
    with pytest.raises(ValueError):
        _native.size_query("hg_spmm_workspace", 100, 0, 10, 1, 1, 0)


def test_library_is_sm100a():
    import subprocess

    lib = ROOT / "paper_2411_01109_b200" / "libhalfgnn.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_reduction_validation():
    from paper_2411_01109_b200.kernels import Reduction

    assert (Reduction().scaling, Reduction().norm) == ("post", "none")
    for bad in ("POST", "mid", ""):
        with pytest.raises(ValueError):
            Reduction(bad, "none")
    with pytest.raises(ValueError):
        Reduction("post", "rows")
    with pytest.raises(ValueError, match="degree norm"):
        Reduction("discretized", "none")


def test_simt_tables():
    from paper_2411_01109_b200 import simt

    assert [simt.warp_load_bytes(w) for w in ("half", "half2", "half4", "half8")] == [64, 128, 256, 512]
    assert simt.sddmm_reduction_rounds(32, "half2") == 4
    assert simt.sddmm_reduction_rounds(32, "half8") == 2
    assert simt.subwarp_layout(16).subwarps == 4 and simt.subwarp_layout(128).subwarps == 1
    assert simt.intra_cta_rounds(8) == 3
    with pytest.raises(ValueError):
        simt.intra_cta_rounds(6)
    with pytest.raises(ValueError):
        simt.warp_load_bytes("half3")


def test_schedules_and_metrics_host():
    from paper_2411_01109_b200 import simt, sparse as sp

    rows = np.arange(130, dtype=np.int64)
    g = sp.CooGraph(131, rows, rows + 1)
    s = simt.plan_edge_parallel(g, 128, 4)
    assert s.num_warps == 2 and s.num_ctas == 1
    simt.check_spmm_rules(g, s)
    m = simt.edge_metrics(g, s, 32, "half2", False)
    assert (m.load_transactions, m.load_bytes, m.staging_writes) == (70, 5 * 256 + 65 * 128, 1)
    with pytest.raises(ValueError):
        simt.plan_edge_parallel(g, 62)
    csr = sp.CsrGraph(5, np.array([0, 70, 70, 75, 75, 75]), np.arange(75) % 5)
    vg = simt.plan_vertex_grouped(csr)
    assert vg.group_rows.tolist() == [0, 0, 0, 2]
    assert vg.starts.tolist() == [0, 32, 64, 70] and vg.ends.tolist() == [32, 64, 70, 75]
    g8 = sp.CooGraph(513, np.zeros(512, dtype=np.int64), np.arange(1, 513, dtype=np.int64))
    m8 = simt.edge_metrics(g8, simt.plan_edge_parallel(g8, 64, 8), 4, "half2", False)
    assert m8.intra_cta_rounds == 3


def test_containers_and_file_format(tmp_path):
    from paper_2411_01109_b200 import sparse as sp

    with pytest.raises(ValueError, match="sorted"):
        sp.CooGraph(3, np.array([1, 0]), np.array([0, 1]))
    with pytest.raises(ValueError, match="positive"):
        sp.CooGraph(0, np.zeros(0), np.zeros(0))
    with pytest.raises(ValueError):
        sp.CsrGraph(2, np.array([0, 2, 1]), np.array([0]))
    t = sp.DenseTensor(np.arange(12, dtype=np.float16).reshape(3, 4))
    p = tmp_path / "t.hsdt"
    sp.save_tensor(t, p)
    raw = p.read_bytes()
    assert raw[:4] == b"HSDT" and len(raw) == 16 + 24
    back = sp.load_tensor(p)
    assert back.mode == "half" and np.array_equal(back.data, t.data)
    p.write_bytes(raw[:-2])
    with pytest.raises(ValueError, match="payload"):
        sp.load_tensor(p)
    padded = sp.pad_features(sp.DenseTensor(np.ones((2, 6), np.float16)), 4)
    assert padded.cols == 8 and not padded.data[:, 6:].any()
    with pytest.raises(ValueError):
        sp.pad_features(t, 3)


def test_partition_split_points_match_restatement():
    import torch

    from paper_2411_01109_b200.partition import remap_to_padded, split_points

    rng = np.random.default_rng(2)
    for _ in range(30):
        deg = rng.integers(0, 30, int(rng.integers(1, 300)))
        deg[int(rng.integers(0, deg.size))] += int(rng.integers(0, 4000))
        off = np.r_[0, np.cumsum(deg)].astype(np.int64)
        for parts in (1, 2, 4, 8):
            np.testing.assert_array_equal(split_points(torch.from_numpy(off), parts),
                                          O.partition_splits(off, parts))
    splits = np.array([0, 3, 3, 7, 10])
    ids = torch.arange(10, dtype=torch.int32)
    got = remap_to_padded(ids, splits, 4).tolist()
    assert got == [0, 1, 2, 8, 9, 10, 11, 12, 13, 14]


def test_operators_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2411_01109_b200 import kernels as K, sparse as sp

    g = sp.CooGraph(3, np.array([0]), np.array([1]))
    x = sp.DenseTensor(np.ones((3, 4), np.float16))
    with pytest.raises(Exception):
        K.spmm_v(g, x)
    with pytest.raises(Exception):
        sp.CooGraph.from_edges(3, [0, 1], [1, 2])


def test_resolve_grad_scale():
    from paper_2411_01109_b200.models import resolve_grad_scale

    assert resolve_grad_scale(1.0, 10) == 1.0
    assert resolve_grad_scale("auto", 2708) == 32.0
    assert resolve_grad_scale("auto", 232_965) == 2048.0
    assert resolve_grad_scale("auto", 10) == 1.0
    assert resolve_grad_scale(256, 5) == 256.0
    for bad in (0.5, 3.0, -2.0):
        with pytest.raises(ValueError, match="power of two"):
            resolve_grad_scale(bad, 100)


@pytest.mark.parametrize("pack_edges", [0, 7, 64, 512])
def test_schedule_pack_restatement_covers_rows_once(pack_edges):
    """The oracle's hg_schedule_build restatement with packs: every row is in
    exactly one whole-row unit, split row or pack; packs are aligned blocks of
    16 rows within the edge budget; units never name a packed row."""
    import numpy as np

    import oracle as O

    rng = np.random.default_rng(pack_edges)
    n = 1003
    deg = rng.choice([0, 0, 1, 2, 5, 40, 700], size=n)
    off = np.r_[0, np.cumsum(deg)].astype(np.int64)
    units, split_rows, slots, packs = O.schedule_units(off, 512, 16, pack_edges)
    cover = np.zeros(n, np.int64)
    np.add.at(cover, units[:, 0][units[:, 3] < 0], 1)
    np.add.at(cover, split_rows[:, 0], 1)
    for r0, beg, end, cnt in packs:
        assert r0 % 16 == 0 and cnt == min(16, n - r0)
        assert beg == off[r0] and end == off[r0 + cnt] and end - beg <= pack_edges
        cover[r0:r0 + cnt] += 1
    assert (cover == 1).all()
    assert slots == sum(-(-d // 512) for d in deg if d > 512)
