"""The C-ABI library loads and exports every symbol include/sivf.h declares;
host-only entry points behave (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "sivf.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sivf_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    so = os.path.join(ROOT, "paper_2601_11808_b200", "lib", "libsivf.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-C", ROOT, "sivf"])
    import paper_2601_11808_b200 as S

    return S.lib()


def test_header_declares_the_contract():
    names = _declared()
    for n in ("sivf_create", "sivf_train_centroids", "sivf_insert", "sivf_delete", "sivf_search",
              "sivf_sliding_window_step", "sivf_merge_topk", "sivf_reclaim", "sivf_dump_state", "sivf_stats"):
        assert n in names


def test_every_declared_symbol_is_exported(L):
    import paper_2601_11808_b200 as S

    for n in _declared():
        assert hasattr(L, n), f"libsivf.so does not export {n}"
        assert n in S.EXPORTS, f"binding does not declare {n}"


def test_arena_bytes_and_validation(L):
    import paper_2601_11808_b200 as S

    c = S.Config()
    c.dim, c.nlist, c.id_capacity, c.num_slabs = 128, 1024, 1_200_000, 46_024
    c.max_batch, c.max_queries, c.max_k, c.max_nprobe = 10_000, 10_000, 128, 128
    c.shard_rank, c.shard_count = 0, 1
    n = ctypes.c_size_t()
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == 0
    payload = 46_024 * 32 * 128 * (4 + 2)  # fp32 slabs + their fp16 scan records
    partial = 10_000 * 128 * 128 * 8  # per-(query, probe) top-k scratch at the max_* limits
    assert payload + partial < n.value < (payload + partial) * 1.3
    full = n.value
    c.flags = S.CFG_NO_SCAN_COPY  # no scan records: exactly 46,024 x (32 x 128 x 2 + 256) bytes less
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == 0
    assert full - n.value == 46_024 * (32 * 128 * 2 + 256)  # fp16 copy + the records' norm and id copies
    c.flags = S.CFG_SPLIT_COPY  # split-fp16 copy at dim 128: 2 x 2 B per value + a scale per slot, no fp16 records
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == 0
    assert n.value > full
    c.flags = 8  # unknown flag bit
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == -1
    c.flags = 0
    c.max_k = 129
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == -1
    c.max_k, c.shard_rank, c.shard_count = 10, 2, 2
    assert L.sivf_arena_bytes(ctypes.byref(c), ctypes.byref(n)) == -1
    assert L.sivf_rc_string(-3) == b"arena too small or misaligned"


def test_no_oracle_in_product_path():
    """The product package never imports, links or loads the oracle."""
    pkg = os.path.join(ROOT, "paper_2601_11808_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "sivf_oracle" not in txt and "import oracle" not in txt and "from oracle" not in txt, f
    so = os.path.join(pkg, "lib", "libsivf.so")
    if os.path.exists(so):
        out = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
        assert "or_" not in " ".join(l.split()[-1] for l in out.splitlines() if l.split()[-1].startswith("or_"))


def test_python_constants_match_the_header():
    """OPT_* / CFG_* in the binding equal the SIVF_OPT_* / SIVF_CFG_* values of include/sivf.h."""
    import re

    import paper_2601_11808_b200 as S

    hdr = open(os.path.join(ROOT, "include", "sivf.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"SIVF_(OPT_[A-Z_]+|CFG_[A-Z_]+)\s*=\s*(\d+)", hdr)}
    assert vals, "no SIVF_OPT_/SIVF_CFG_ enumerators found"
    for name, v in vals.items():
        assert getattr(S, name) == v, f"{name}: binding {getattr(S, name, None)} header {v}"
