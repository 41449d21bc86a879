"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/bspmm.h declares, rejects bad arguments, and its host-only functions
(partition, subWarp rule, planner) agree with the oracle / the paper.
No compute call touches a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_1903_11409_b200 as bs
from paper_1903_11409_b200 import _lib


def test_exports_every_header_symbol():
    syms = bs.header_symbols()
    assert len(syms) >= 18, syms
    raw = ctypes.CDLL(bs.LIB_PATH)
    missing = [s for s in syms if not hasattr(raw, s)]
    assert not missing, missing
    # nothing else leaks: every exported function is a declared bspmm_* entry point
    import subprocess
    dyn = subprocess.run(["nm", "-D", "--defined-only", bs.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in dyn.splitlines() if " T " in ln}
    ours = {x for x in exported if x.startswith("bspmm_")}
    assert ours == set(syms), (ours ^ set(syms))
    assert not [x for x in exported if "bspmm" in x and not x.startswith("bspmm_")]


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", bs.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_status_strings_and_null_handle():
    lib = _lib.lib
    assert lib.bspmm_status_string(0) == b"BSPMM_SUCCESS"
    assert lib.bspmm_status_string(4) == b"BSPMM_ERROR_INDEX"
    assert lib.bspmm_destroy(None) == 0
    assert lib.bspmm_csr(None, 1, 1, None, None, None, None, None, None, 1, None, 1) == _lib.INVALID_VALUE
    assert lib.bspmm_sync(None) == _lib.INVALID_VALUE
    assert lib.bspmm_launch_count(None) == -1


def test_create_without_gpu_is_not_supported_or_ok():
    h = ctypes.c_void_p()
    assert _lib.lib.bspmm_create(None, 0, None, 0) == _lib.INVALID_VALUE
    assert _lib.lib.bspmm_create(ctypes.byref(h), 0, None, 0x80) == _lib.INVALID_VALUE
    st = _lib.lib.bspmm_create(ctypes.byref(h), 0, None, 0)
    import torch
    if not torch.cuda.is_available():
        assert st == _lib.NOT_SUPPORTED and not h.value
    else:
        assert st == _lib.SUCCESS
        _lib.lib.bspmm_destroy(h)


def test_subwarp_rule_golden(golden):
    for n_b, want in golden["subwarp"]["cases"]:
        assert bs.subwarp(n_b) == want, (n_b, golden["subwarp"]["cite"])
    assert bs.subwarp(0) == 0
    # invariants: power of two, monotone, 32 above 16
    prev = 0
    for n in range(1, 300):
        s = bs.subwarp(n)
        assert s & (s - 1) == 0 and s >= prev and s >= min(n, 32) and (n <= 16 or s == 32)
        prev = s


def test_partition_matches_oracle_bit_exact(golden):
    for ex in golden["partition"]:
        nnz_off = np.concatenate([[0], np.cumsum(ex["nnz"])]).astype(np.int64)
        assert list(bs.partition(nnz_off, ex["k"], ex["parts"])) == ex["split"], ex["cite"]
    rng = np.random.default_rng(11)
    for _ in range(2000):
        batch = int(rng.integers(0, 60))
        nnz_off = np.concatenate([[0], np.cumsum(rng.integers(0, 40, size=batch))]).astype(np.int64)
        k, G = int(rng.integers(1, 1025)), int(rng.integers(1, 9))
        assert np.array_equal(bs.partition(nnz_off, k, G), oracle.partition(nnz_off, k, G))


def test_partition_c5_shape():
    import synth
    n, z = synth.counts(synth.MOL, (20, 60, 0, 0), synth.BASE_SEED + 5, 0, 65536)
    nnz_off = np.concatenate([[0], np.cumsum(z)]).astype(np.int64)
    for G in (1, 2, 4, 8):
        s = bs.partition(nnz_off, 256, G)
        assert np.array_equal(s, oracle.partition(nnz_off, 256, G))
        cost = [int(nnz_off[s[r + 1]] - nnz_off[s[r]]) for r in range(G)]
        assert max(cost) - min(cost) <= 2 * int(z.max())         # within a graph or two


def test_partition_rejects_bad_args():
    with pytest.raises(bs.BspmmError):
        bs.partition(np.array([0, 5, 3], dtype=np.int64), 4, 2)      # non-monotone
    with pytest.raises(bs.BspmmError):
        bs.partition(np.array([0, 5], dtype=np.int64), 4, 0)


@pytest.mark.parametrize("k", [1, 3, 4, 5, 16, 17, 33, 64, 128, 256, 512, 1000, 1024, 4096])
@pytest.mark.parametrize("batch", [1, 4, 100, 200, 65536])
def test_plan_invariants(k, batch):
    for aligned in (True, False):
        if aligned and k % 4:
            continue
        for rows in (0, 8, 60, 300, 5000):
            p = bs.plan(k, batch, aligned=aligned, max_rows=rows)
            assert p["tiles"] == -(-k // p["kt"])                            # tiles cover [0, k)
            assert p["kt"] * (p["tiles"] - 1) < k <= p["kt"] * p["tiles"]    # disjoint, no empty tile
            cols = -(-p["kt"] // 4) if p["vec"] else p["kt"]
            pref = 4 if (p["vec"] and p["kt"] >= 128 and p["units"] <= 4 * 148) else 2
            assert p["lanes"] == bs.subwarp(-(-cols // pref))                # PAPER.md:150-155 on chunks
            assert p["lanes"] * p["chunks"] >= cols and p["chunks"] in (1, 2, 4)
            p1 = bs.plan(k, batch, aligned=aligned, max_rows=rows, chunks=1)
            assert p1["lanes"] == bs.subwarp(cols)                           # the paper's rule, 1 chunk/lane
            assert p["smem_bytes"] <= 232448 and p["stages"] >= 1
            assert p["units"] == batch * p["tiles"]
            assert 1 <= p["grid"] <= min(p["units"], 148)
            assert p["threads"] == 32 * (1 + (15 if p["chunks"] == 4 else 16))
            if aligned:
                assert p["kt"] % 4 == 0
            if rows and rows * p["kt"] * 4 <= 100000:
                assert p["stage_b_bytes"] >= rows * p["kt"] * 4                 # fits -> staged


def test_plan_paper_shapes():
    # C4 (PAPER.md:366 shape): 100 whole matrices occupy 100 of 148 SMs -- more
    # than half, so no column blocking (several units per CTA cost more than
    # idle SMs, DESIGN.md §3 planner); two stages of 50 x 512 tiles fit
    p = bs.plan(512, 100, max_rows=50)
    assert p["tiles"] == 1 and p["units"] == 100 and p["stages"] >= 2
    # 16 such matrices would leave most SMs idle -> column blocking until <= 32 KB tiles
    p = bs.plan(512, 16, max_rows=50)
    assert p["tiles"] > 1 and 50 * p["kt"] * 4 <= 32768
    # C5: whole rows, one unit per matrix
    p = bs.plan(256, 65536, max_rows=60)
    assert p["tiles"] == 1 and p["stages"] >= 2


def test_multimem_store_sass():
    """The multicast-store kernel variant (EPI = 2, NEXT-4b) writes C with the
    same 128-bit STG as the plain kernel minus the evict-first hint: on sm_100a
    multimem.st is an ordinary store whose fan-out comes from the multicast VA
    mapping.  This is what lets the GPU tests check that variant by unicast
    emulation where the driver refuses multicast objects."""
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None and not os.path.exists("/usr/local/cuda/bin/cuobjdump"):
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

    sass = subprocess.run([exe, "-sass", bs.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)

    def stores(prefix):  # 128-bit global stores of the CSR-mode kernel <CH=2, VEC, EPI=..., COO=0, ONE=0>
        body = [f for f in funcs if f.startswith(prefix)]
        assert len(body) == 1, (prefix, len(body))
        return set(re.findall(r"\bSTG\.E[.A-Z0-9]*\.128\b", body[0]))

    mc = stores("_ZN5bspmm15spmm_csr_kernelILi2ELb1ELi2ELb0ELb0EE")
    plain = stores("_ZN5bspmm15spmm_csr_kernelILi2ELb1ELi0ELb0ELb0EE")
    assert mc == {"STG.E.128"}, mc
    assert plain == {"STG.E.EF.128"}, plain


def test_gcn_sass_uses_tcgen05():
    """The fused layer's kernel issues tensor-core MMAs (UTCHMMA), TMEM loads
    (LDTM) and tensor TMA (UTMALDG) -- checked in the shipped library."""
    import os
    import subprocess
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1903_11409_b200", "libbspmm.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    i = out.find("gcn_fused_kernel")
    assert i >= 0
    body = out[i:out.find("Function :", i + 20)]
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "UTCBAR"):
        assert mnem in body, mnem


def test_gcn_cta_pair_sass():
    """The CTA-pair instantiation of the fused layer issues the 2-SM MMA
    (UTCHMMA.2CTA), its multicast commit (UTCBAR.2CTA.MULTICAST), 2-SM tensor
    TMA (UTMALDG.2D.2CTA) and the pair TMEM allocation."""
    import os
    import re
    import subprocess
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1903_11409_b200", "libbspmm.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    m = re.search(r"Function : \S*gcn_fused_kernelILi2ELi2E", out)
    assert m, "no CTA-pair instantiation of gcn_fused_kernel"
    body = out[m.start():out.find("Function :", m.start() + 20)]
    for mnem in ("UTCHMMA.2CTA", "UTCBAR.2CTA.MULTICAST", "UTMALDG.2D.2CTA", "UTCATOMSWS.2CTA"):
        assert mnem in body, mnem


def test_hot_kernels_do_not_spill():
    """The CSR pipeline's plain-store instantiations (the bench path), the tile
    kernel and the fused GCN kernel keep everything in registers: a code change
    that makes them spill (a 19% C5 regression once, from one added prologue
    line) fails here, on the CPU, before any GPU time is spent."""
    import os
    import re
    import subprocess
    lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1903_11409_b200",
                       "libbspmm.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--dump-resource-usage", lib], capture_output=True,
                         text=True).stdout
    funcs = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out)
    hot = [(f, int(st)) for f, _, st in funcs
           if re.search(r"spmm_csr_kernelILi[124]ELb1ELi0ELb0E", f) or "spmm_tile_kernel" in f or "gcn_fused" in f]
    assert len(hot) >= 6, hot
    assert all(st == 0 for _, st in hot), [f for f, st in hot if st]
