"""Multi-process exchange with the PRODUCT engine on one GPU.

World-size 2 / 3 / 4 jobs of separate processes that all drive cuda:0 with
CudaEngine (every encode / decode is a sm_100a kernel through the C ABI); the
collectives run over gloo with host staging (comm.all_gather_flat & co.), so the
full multi-rank logic — row shards with remainder, fixed-size wire slots, per-peer
step counters, own shard = sender.base, batched K2 over peers — executes with
real device codecs on a 1-GPU box.  Every rank's reconstruction must equal the
numpy simulation of the reference mesh (mesh.py:188-237: per-shard sender channel,
receivers mirror senders, full = vstack) bit for bit after EVERY step, and all
ranks' blake2b digests must agree (mesh:237, 320-324).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu

STEPS = 5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spec(name):
    from paper_2507_17511_b200 import compressors as cx

    if name == "topk":
        return cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=0.05)
    if name == "nm2:4":
        return cx.CompressorSpec(cx.CompressorKind.NM_BLOCK, n=2, m=4)
    return cx.CompressorSpec(cx.CompressorKind(name))


def _ocodec(name):
    if name == "topk":
        return O.Codec(O.TOPK, keep_fraction=0.05)
    if name == "nm2:4":
        return O.Codec(O.NMBLOCK, nm=(2, 4))
    if name == "identity":
        return O.Codec(O.RAW)
    return O.Codec({"sign1bit": O.SIGN1, "quant2bit": O.QUANT2}[name])


def _inputs(rows, cols, seed=99):
    return synth.flux_like(rows, cols, STEPS, seed=seed)


def _init(rank, world, port, backend):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0  # gloo: every rank shares cuda:0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_patch(rank, world, port, rows, cols, codec, mode, topology, out_dir, backend="gloo"):
    _init(rank, world, port, backend)
    try:
        from paper_2507_17511_b200 import _lib
        from paper_2507_17511_b200.comm import CudaEngine, PatchParallelExchange, RingExchange

        cls = RingExchange if topology == "ring" else PatchParallelExchange
        ex = cls(rows, cols, _spec(codec), mode=mode, warmup=1, in_dtype=torch.bfloat16)
        assert isinstance(ex.engine, CudaEngine)
        n0 = _lib.load().cc_launch_count()
        fulls, digests = [], []
        for x in _inputs(rows, cols):
            xd = torch.from_numpy(x[ex.lo:ex.hi]).cuda().to(torch.bfloat16)
            ex.step(xd)
            fulls.append(ex.reconstruction().cpu().numpy())
            digests.append(ex.digest())
        torch.cuda.synchronize()
        assert _lib.load().cc_launch_count() - n0 >= 2 * STEPS  # device codecs did the work
        np.save(os.path.join(out_dir, f"full{rank}.npy"), np.stack(fulls))
        with open(os.path.join(out_dir, f"dig{rank}.bin"), "wb") as f:
            f.write(b"".join(digests))
    finally:
        dist.destroy_process_group()


def _simulate_mesh(world, rows, cols, codec, mode, seed=99):
    """The reference mesh's all-gather semantics on the numpy oracle: per step the
    vstack of every shard's sender base (receivers mirror senders bit-exactly)."""
    bounds = O.shard_rows(rows, world)
    oc = _ocodec(codec)
    chans = [O.Channel(mode, 1, np.zeros((hi - lo, cols), np.float32)) for lo, hi in bounds]
    rcv = [O.Channel(mode, 1, np.zeros((hi - lo, cols), np.float32)) for lo, hi in bounds]
    out = []
    for t, x in enumerate(_inputs(rows, cols, seed), start=1):
        for (lo, hi), ch, rc in zip(bounds, chans, rcv):
            tag, body, _ = O.send(ch, x[lo:hi], oc)
            O.receive(rc, t, t <= 1, tag, body, oc)
            assert np.array_equal(rc.base, ch.base)
        out.append(np.vstack([ch.base for ch in chans]))
    return np.stack(out)


def _run_patch(world, rows, cols, codec, mode="residual_with_feedback", topology="allgather", backend="gloo"):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_patch, args=(world, _free_port(), rows, cols, codec, mode, topology, d, backend),
                 nprocs=world, join=True)
        fulls = [np.load(os.path.join(d, f"full{r}.npy")) for r in range(world)]
        digs = [open(os.path.join(d, f"dig{r}.bin"), "rb").read() for r in range(world)]
    assert all(dg == digs[0] for dg in digs), "ranks diverged (mesh:320-324)"
    ref = _simulate_mesh(world, rows, cols, codec, mode)
    for r, f in enumerate(fulls):
        for t in range(STEPS):
            assert f[t].tobytes() == ref[t].tobytes(), f"rank {r} step {t + 1} != reference mesh"


# FLUX-width rows take the persistent fused K1; the ragged 37 x 64 shape takes the
# multi-kernel path with a remainder shard
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("codec", ["quant2bit", "sign1bit"])
def test_patch_allgather_cuda_engine_flux_width(world, codec):
    _run_patch(world, 24 * world + 5, 3072, codec)


@pytest.mark.parametrize("codec", ["quant2bit", "topk", "nm2:4", "identity"])
def test_patch_allgather_cuda_engine_ragged(codec):
    _run_patch(2, 37, 64, codec)


def test_patch_allgather_cuda_engine_naive_world4():
    _run_patch(4, 64, 384, "quant2bit", mode="naive")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("codec", ["quant2bit", "topk"])
def test_ring_cuda_engine(world, codec):
    """Ring hops (bodies forwarded verbatim, origin (rank - hop) % P) rebuild exactly
    the all-gather reconstruction (mesh:214-229 with the origin fixed)."""
    _run_patch(world, 16 * world + 3, 3072, codec, topology="ring")


def _worker_ulysses(rank, world, port, n_local, cols, codec, out_dir, backend="gloo"):
    _init(rank, world, port, backend)
    try:
        from paper_2507_17511_b200.comm import UlyssesAllToAll

        ex = UlyssesAllToAll(n_local, cols, _spec(codec), in_dtype=torch.bfloat16)
        outs = []
        for x in _inputs(world * n_local, cols, seed=7):
            xd = torch.from_numpy(x[rank * n_local:(rank + 1) * n_local]).cuda().to(torch.bfloat16)
            outs.append(ex.step(xd).cpu().numpy())
        np.save(os.path.join(out_dir, f"u{rank}.npy"), np.stack(outs))
        with open(os.path.join(out_dir, f"seg{rank}"), "w") as f:
            f.write(str(int(ex.segmented)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cols,codec", [(2, 3072, "sign1bit"), (4, 3072, "sign1bit"), (2, 3072, "quant2bit"),
                                              (2, 256, "sign1bit"), (2, 3072, "identity")])
def test_ulysses_cuda_engine(world, cols, codec):
    _run_ulysses(world, cols, codec)


def _run_ulysses(world, cols, codec, backend="gloo"):
    """Composed parity: every directed (src, dst) chunk is its own
    channel; rank dst holds the vstack over src of those channels' bases."""
    n_local = 24
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_ulysses, args=(world, _free_port(), n_local, cols, codec, d, backend), nprocs=world,
                 join=True)
        outs = [np.load(os.path.join(d, f"u{r}.npy")) for r in range(world)]
        seg = [open(os.path.join(d, f"seg{r}")).read() for r in range(world)]
    if cols == 3072 and codec != "identity":
        assert seg == ["1"] * world  # the one-launch segmented K1 was exercised
    cw = cols // world
    oc = _ocodec(codec)
    chans = {(s, t): O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n_local, cw), np.float32))
             for s in range(world) for t in range(world)}
    for step, x in enumerate(_inputs(world * n_local, cols, seed=7)):
        for s in range(world):
            for t in range(world):
                O.send(chans[(s, t)], x[s * n_local:(s + 1) * n_local, t * cw:(t + 1) * cw], oc)
        for t in range(world):
            exp = np.vstack([chans[(s, t)].base for s in range(world)])
            assert outs[t][step].tobytes() == exp.tobytes(), f"dst {t} step {step + 1}"
