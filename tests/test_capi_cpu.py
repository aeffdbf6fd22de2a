"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
symbol include/mhlmoe.h declares, and its pure-host plan logic (validation,
HP head partition, k-independent all-to-all bytes) is right.  No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "mhlmoe.h")).read()
    return sorted(set(re.findall(r"^MHL_API\s+[\w\s\*]+?\b(\w+)\(", src, flags=re.M)))


def test_library_loads_and_exports_header_symbols():
    from paper_2602_04870_b200 import mhlmoe as C
    syms = _header_symbols()
    assert len(syms) >= 12
    lib = C.library()
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(C.EXPORTS)
    # the exported dynamic symbol table holds exactly the ABI (internal kernels are hidden)
    out = os.popen(f"nm -D --defined-only {C.LIB_PATH}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(syms)


def test_library_is_sm100a():
    from paper_2602_04870_b200 import mhlmoe as C
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {C.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def _q(**kw):
    from paper_2602_04870_b200 import mhlmoe as C
    base = dict(T_loc=256, d=64, N_h=4, d_h=16, N_e=8, k=2, d_e=16, dtype="fp32", world_size=1, rank=0, flags=0)
    base.update(kw)
    return C.hp_plan_query(C.make_config(**base))


@pytest.mark.parametrize("kw,status", [
    (dict(k=0), "MHL_ERR_CONFIG"), (dict(k=9), "MHL_ERR_CONFIG"),
    (dict(world_size=3), "MHL_ERR_CONFIG"), (dict(world_size=8), "MHL_ERR_CONFIG"),
    (dict(T_loc=0), "MHL_ERR_CONFIG"), (dict(rank=2, world_size=2), "MHL_ERR_CONFIG"),
    (dict(d_h=12), "MHL_ERR_UNSUPPORTED"), (dict(N_e=32, k=17), "MHL_ERR_UNSUPPORTED"),
])
def test_plan_query_rejects_bad_configs(kw, status):
    from paper_2602_04870_b200 import mhlmoe as C
    with pytest.raises(C.MhlError) as ei:
        _q(**kw)
    assert C.STATUS[ei.value.status] == status
    assert C.mhl_last_error()


def test_plan_query_hp_partition_and_bytes():
    for G in (1, 2, 4, 8):
        heads = []
        for r in range(G):
            info = _q(T_loc=65536, d=2048, N_h=8, d_h=256, N_e=64, k=8, d_e=128, dtype="bf16", world_size=G, rank=r)
            heads.append((info["head_begin"], info["head_end"]))
            assert info["tokens_global"] == 65536 * G
            assert info["a2a_bytes_per_peer"] == 65536 * (8 // G) * 256 * 2
            assert info["a2a_bytes_per_rank"] == info["a2a_bytes_per_peer"] * (G - 1)
        assert heads == [(r * 8 // G, (r + 1) * 8 // G) for r in range(G)]
    # k-independent bytes: only the workspace grows with k
    infos = [_q(T_loc=4096, d=2048, N_h=8, d_h=256, N_e=64, k=k, d_e=128, dtype="bf16", world_size=4, rank=1)
             for k in (2, 4, 8, 16)]
    assert len({i["a2a_bytes_per_rank"] for i in infos}) == 1
    assert infos[0]["workspace_bytes"] < infos[-1]["workspace_bytes"]


def test_status_strings():
    from paper_2602_04870_b200 import mhlmoe as C
    for s, name in C.STATUS.items():
        assert C.mhl_status_string(s) == name


def test_oracle_is_not_imported_by_the_product():
    """The product path must never route through the oracle (or any CPU fallback)."""
    for dirpath, _d, files in os.walk(os.path.join(ROOT, "paper_2602_04870_b200")):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).lower().replace("oracle/", ""), f


def test_score_matrix_never_materialised_memory_flat_in_N_e():
    """Fig. 4 / P:1277 and north_star: the fused router never writes the T x N_e score matrix.  The
    plan's device memory (saved + workspace) has per-expert tables and per-replica buffers, but no
    T*N_e term of score size: doubling T adds far less than the naive router's extra score bytes
    for N_e = 1536 vs 64 experts."""
    def mem(T, N_e):
        i = _q(T_loc=T, d=1024, N_h=8, d_h=128, N_e=N_e, k=4, d_e=128, dtype="bf16")
        return i["saved_bytes"] + i["workspace_bytes"]
    cross = (mem(32768, 1536) - mem(32768, 64)) - (mem(16384, 1536) - mem(16384, 64))
    naive = 8 * 16384 * (1536 - 64) * 4          # fp32 scores of 16384 more tokens x 1472 more experts
    assert cross < 0.1 * naive, (cross, naive)


def test_routing_tokens_plan_doubles_the_scatter_only():
    """separate routing sub-tokens double the HP scatter volume; the plan's byte counts say
    so (the gather of head outputs is unchanged, see mhl_a2a_bytes_posted)."""
    from paper_2602_04870_b200 import mhlmoe as C
    for G in (2, 4, 8):
        a = _q(T_loc=4096, d=2048, N_h=8, d_h=256, N_e=64, k=8, d_e=128, dtype="bf16", world_size=G, rank=0)
        b = _q(T_loc=4096, d=2048, N_h=8, d_h=256, N_e=64, k=8, d_e=128, dtype="bf16", world_size=G, rank=0,
               flags=C.MHL_FLAG_ROUTING_TOKENS)
        assert b["a2a_bytes_per_peer"] == 2 * a["a2a_bytes_per_peer"]
        assert b["a2a_bytes_per_rank"] == 2 * a["a2a_bytes_per_rank"]


def test_fused_combine_flag_is_rejected():
    """The in-kernel combine experiment (MHL_FLAG_FUSED_COMBINE) was removed (measured slower, and it
    needed every CTA resident for its cross-CTA spin); the flag is refused before any launch."""
    from paper_2602_04870_b200 import mhlmoe as C
    cfg = C.make_config(1024, 256, 2, 128, 64, 8, 64, "bf16", 1, 0, C.MHL_FLAG_FUSED_COMBINE)
    try:
        C.hp_plan_query(cfg)
    except C.MhlError as e:
        assert C.STATUS[e.status] == "MHL_ERR_UNSUPPORTED"
    else:
        raise AssertionError("MHL_FLAG_FUSED_COMBINE accepted")


def test_det_dp_flag_validation():
    """MHL_FLAG_DET_DP needs T_loc a power-of-two multiple of 8192 and G a power of two."""
    from paper_2602_04870_b200 import mhlmoe as C
    ok = C.make_config(16384, 256, 4, 64, 16, 4, 64, "bf16", 2, 0, C.MHL_FLAG_DET_DP)
    C.hp_plan_query(ok)
    for T_loc, G in ((12288, 1), (24576, 1), (8192, 3)):
        cfg = C.make_config(T_loc, 256, 6 if G == 3 else 4, 64, 16, 4, 64, "bf16", G, 0, C.MHL_FLAG_DET_DP)
        try:
            C.hp_plan_query(cfg)
        except C.MhlError as e:
            assert C.STATUS[e.status] == "MHL_ERR_UNSUPPORTED"
        else:
            raise AssertionError((T_loc, G))


def test_require_tc_flag_refuses_simt_fallback_shapes():
    """MHL_FLAG_REQUIRE_TC: a shape some step has no tcgen05 kernel for is refused up front (pure host),
    a fully supported one (the paper head) is accepted."""
    from paper_2602_04870_b200 import mhlmoe as C
    C.hp_plan_query(C.make_config(1024, 512, 2, 256, 64, 8, 128, "bf16", 1, 0, C.MHL_FLAG_REQUIRE_TC))
    for (d_h, N_e, k, d_e, dt) in ((256, 16, 4, 128, "bf16"), (192, 64, 8, 64, "bf16"), (32, 16, 4, 32, "bf16"),
                                   (256, 64, 8, 128, "fp32")):
        cfg = C.make_config(1024, 2 * d_h, 2, d_h, N_e, k, d_e, dt, 1, 0, C.MHL_FLAG_REQUIRE_TC)
        try:
            C.hp_plan_query(cfg)
        except C.MhlError as e:
            assert C.STATUS[e.status] == "MHL_ERR_UNSUPPORTED"
        else:
            raise AssertionError((d_h, N_e, k, d_e, dt))


def test_bwd_fused_flag_matches_header_and_is_accepted():
    """MHL_FLAG_BWD_FUSED (the one-kernel expert backward input side) is the header's value and a
    plan query accepts it on a supported and on an unsupported shape (the latter falls back to the
    two-kernel path, which mhl_kernel_paths reports on the GPU)."""
    import re
    from paper_2602_04870_b200 import mhlmoe as C
    hdr = open(os.path.join(ROOT, "include", "mhlmoe.h")).read()
    m = re.search(r"#define MHL_FLAG_BWD_FUSED (\d+)u", hdr)
    assert m and int(m.group(1)) == C.MHL_FLAG_BWD_FUSED
    assert C.PATHS["expert_bwd_fused"] == 1 << 15 and "MHL_PATH_EXPERT_BWD_FUSED (1u << 15)" in hdr
    for d_e in (128, 256):   # 2 d_e + d_h <= 512 only for d_e = 128
        C.hp_plan_query(C.make_config(1024, 512, 2, 256, 64, 8, d_e, "bf16", 1, 0, C.MHL_FLAG_BWD_FUSED))
