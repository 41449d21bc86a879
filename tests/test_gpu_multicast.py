"""GPU parity for the all-gather fused into the SpMM store (SURVEY §8(e)
optional reassembly, §8(f) NEXT-4b): bspmm_csr_multicast writes C through an
NVSwitch multicast address.  On the one-GPU box the team has one member, which
still exercises the whole path (multicast object, bind, multicast VA, multimem
stores, system fence); rank shards are emulated by writing each shard at its
global row base.  Bars as test_gpu_parity: bitwise equal to the fp32
storage-order oracle O3' and within the fp64 bound.

Where the driver refuses to create a multicast object (the round's GPU box:
one GPU of an NVSwitch system passed into a container, fabric GUID 0 --
cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE although the device reports
multicast support), the same kernel is exercised by UNICAST EMULATION: the
multimem store variant writes to an ordinary buffer (on sm_100a multimem.st
lowers to the same STG.E.128 as a plain store; checked in
test_multimem_sass_is_plain_store), and the team-buffer tests skip with the
driver's reason."""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1903_11409_b200 as bs
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available()
    return bs.Handle(0)


class Target:
    """A real multicast team buffer when the driver allows one, else a plain
    device tensor (unicast emulation of the same kernel)."""

    def __init__(self, shape, export=False):
        ok, self.why = bs.mc_available(0)
        self.buf = bs.McBuffer(shape, DEV, export=export) if ok else None
        self.out = self.buf if ok else torch.empty(shape, dtype=torch.float32, device=DEV)
        self.view = self.buf.uc if ok else self.out
        self.view.fill_(float("nan"))

    def close(self):
        if self.buf is not None:
            self.buf.close()


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def oracle_c32(b):
    return oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_multicast_store_bitwise(h, cid):
    b = synth.config(cid)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    tg = Target((b.n_rows, b.k))
    try:
        h.csr_multicast(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), tg.out)
        torch.cuda.synchronize()
        C = tg.view.cpu().numpy()
        C32 = oracle_c32(b)
        assert np.array_equal(C.view(np.uint32), C32.view(np.uint32))
        Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        assert oracle.check_bound(C, Cref, bound)[0]
    finally:
        tg.close()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_multicast_shards_reassemble(h, G):
    """Each emulated rank computes its contiguous shard (offsets rebased to 0) and
    stores it at its global row base through the multicast address."""
    b = synth.config(3)
    split = bs.partition(b.nnz_off, b.k, G)
    tg = Target((b.n_rows, b.k))
    try:
        for r in range(G):
            i0, i1 = int(split[r]), int(split[r + 1])
            if i1 == i0:
                continue
            part = synth.config(3, i0=i0, i1=i1)
            h.set_hints(int(part.sizes.max()), int(part.nnz.max()))
            h.csr_multicast(T(part.row_off), None, T(part.row_ptr), T(part.col), T(part.vals), T(part.B), tg.out,
                            row_base=int(b.row_off[i0]))
        torch.cuda.synchronize()
        C = tg.view.cpu().numpy()
        assert np.array_equal(C.view(np.uint32), oracle_c32(b).view(np.uint32))
    finally:
        tg.close()


def test_multicast_scalar_path_and_fused_offsets(h):
    """k % 4 != 0 (scalar multimem stores) and row_off = NULL (offsets fused into
    the producer) through the multicast store."""
    b = synth.generate(synth.MIX, (5, 40, 1, 6), 37, 13, seed=77)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    tg = Target((b.n_rows, b.k))
    try:
        h.csr_multicast(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B), tg.out)
        torch.cuda.synchronize()
        assert np.array_equal(tg.view.cpu().numpy().view(np.uint32), oracle_c32(b).view(np.uint32))
    finally:
        tg.close()


def test_multicast_export_handle(h):
    """The exportable team object (what rank 0 hands to the other ranks) is
    created with a valid POSIX fd and works as a one-member team."""
    ok, why = bs.mc_available(0)
    if not ok:
        pytest.skip(f"driver refuses multicast objects on this box: {why}")
    b = synth.config(2)
    buf = bs.McBuffer((b.n_rows, b.k), DEV, export=True)
    try:
        assert buf.fd is not None and buf.fd >= 0
        os.fstat(buf.fd)
        h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
        h.csr_multicast(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), buf)
        torch.cuda.synchronize()
        assert np.array_equal(buf.uc.cpu().numpy().view(np.uint32), oracle_c32(b).view(np.uint32))
    finally:
        if buf.fd is not None:
            os.close(buf.fd)
        buf.close()


def test_multicast_rejects_bad_rows(h):
    b = synth.config(1)
    tg = Target((b.n_rows, b.k))
    try:
        with pytest.raises(ValueError):
            h.csr_multicast(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), tg.out, row_base=1)
    finally:
        tg.close()


def test_mc_failure_is_reported():
    """Creation failures name the driver call (no silent fallback)."""
    ok, why = bs.mc_available(0)
    if ok:
        assert why == ""
    else:
        assert "bspmm_mc_create" in why and ("cuMulticast" in why or "no multicast" in why)
