"""The exchanges as C-ABI objects (cc_comm_* / cc_allgather_* / cc_alltoall_*):
one library call = K1 encode -> NCCL collective -> K2 decode.

* world 1: the C all-gather layer equals the Python PatchParallelExchange and the
  oracle (bodies, base, feedback, loopback reconstruction) bit for bit;
* a communicator adopted from PyTorch (ProcessGroupNCCL._comm_ptr) and one built
  from a unique id both drive it;
* a plain C program (tests/c/exchange_demo.c, no Python) runs the step;
* multi-rank: 2 processes on 2 GPUs over NCCL vs the reference mesh (skipped on a
  1-GPU box — tests/test_gpu_multiproc.py covers the Python exchange there).
"""

import os
import socket
import subprocess
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import cc_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)


def _spec(name):
    from paper_2507_17511_b200 import compressors as cx

    if name == "topk":
        return cx.CompressorSpec(cx.CompressorKind.TOPK, keep_fraction=0.05)
    if name == "nm2:4":
        return cx.CompressorSpec(cx.CompressorKind.NM_BLOCK, n=2, m=4)
    if name == "quant4bit-per_token":
        return cx.CompressorSpec(cx.CompressorKind.QUANT4BIT, scale_mode="per_token")
    return cx.CompressorSpec(cx.CompressorKind(name))


def _ocodec(name):
    return {"topk": O.Codec(O.TOPK, keep_fraction=0.05), "nm2:4": O.Codec(O.NMBLOCK, nm=(2, 4)),
            "identity": O.Codec(O.RAW), "sign1bit": O.Codec(O.SIGN1), "quant2bit": O.Codec(O.QUANT2),
            "quant4bit-per_token": O.Codec(O.QUANT4, scale_mode="per_token")}[name]


@pytest.mark.parametrize("codec", ["quant2bit", "sign1bit", "quant4bit-per_token", "topk", "nm2:4", "identity"])
@pytest.mark.parametrize("mode", ["residual_with_feedback", "naive"])
def test_c_allgather_world1_vs_python_and_oracle(codec, mode):
    from paper_2507_17511_b200.comm import CAllGather, PatchParallelExchange

    rows, cols = 96, 3072
    c = CAllGather(rows, cols, _spec(codec), mode=mode)
    py = PatchParallelExchange(rows, cols, _spec(codec), mode=mode, overlap=False)
    och = O.Channel(mode, 1, np.zeros((rows, cols), np.float32))
    for t, x in enumerate(synth.flux_like(rows, cols, 5, seed=11), start=1):
        xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
        rc = c.step(xd)
        rp = py.step(xd)
        torch.cuda.synchronize()
        tag, body, orec = O.send(och, x, _ocodec(codec))
        if t > 1 and codec != "identity":
            assert c.body().cpu().numpy().tobytes() == body, f"body, step {t}"
        assert torch.equal(rc, rp), f"reconstruction != Python exchange, step {t}"
        assert np.array_equal(c.sender_base().cpu().numpy(), och.base), f"base, step {t}"
        assert torch.equal(rc, c.sender_base()), "loopback receiver != sender"
        if mode == "residual_with_feedback":
            assert np.array_equal(c.sender_aux().cpu().numpy(), och.fb), f"feedback, step {t}"
        assert c.record()[0].item() == pytest.approx(orec["compression_error"], rel=1e-6, abs=1e-30)
    c.close()


def test_c_alltoall_world1_vs_oracle():
    from paper_2507_17511_b200.comm import CAllToAll

    n, C = 64, 3072
    a2a = CAllToAll(n, C, _spec("sign1bit"))
    och = O.Channel(O.WITH_FEEDBACK, 1, np.zeros((n, C), np.float32))
    for x in synth.flux_like(n, C, 4, seed=12):
        out = a2a.step(torch.from_numpy(x).cuda().to(torch.bfloat16))
        torch.cuda.synchronize()
        O.send(och, x, O.Codec(O.SIGN1))
        assert np.array_equal(out.cpu().numpy(), och.base)
    a2a.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_comm_from_unique_id_and_from_torch_process_group():
    from paper_2507_17511_b200.comm import CAllGather, CComm

    comm = CComm.init_rank(CComm.unique_id(), 1, 0)
    assert (comm.rank, comm.size) == (0, 1)
    layer = CAllGather(32, 384, _spec("quant2bit"), comm=comm)
    x = torch.from_numpy(synth.flux_like(32, 384, 1, seed=3)[0]).cuda().to(torch.bfloat16)
    layer.step(x)
    torch.cuda.synchronize()
    assert torch.equal(layer.reconstruction(), x.float())  # warmup step: raw, lossless
    layer.close()
    comm.destroy()

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tcomm = CComm.from_process_group()
        assert (tcomm.rank, tcomm.size) == (0, 1)
        layer = CAllGather(32, 384, _spec("quant2bit"), comm=tcomm)
        layer.step(x)
        torch.cuda.synchronize()
        assert torch.equal(layer.reconstruction(), x.float())
        layer.close()
        tcomm.destroy()  # adopted: the process group keeps owning the communicator
        t = torch.ones(4, device="cuda")
        dist.all_reduce(t)  # still usable by torch
        assert t.sum().item() == 4.0
    finally:
        dist.destroy_process_group()


def test_plain_c_program_runs_the_exchange_step():
    libdir = os.path.join(ROOT, "paper_2507_17511_b200", "lib")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "demo")
        subprocess.run(["gcc", "-O2", os.path.join(ROOT, "tests", "c", "exchange_demo.c"), "-I",
                        os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", f"-L{libdir}",
                        "-lcompactcomm_b200", "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", "-o",
                        exe], check=True)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    assert "exchange_demo ok" in r.stdout


def _worker(rank, world, port, uid, rows, cols, codec, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    from paper_2507_17511_b200.comm import CAllGather, CComm

    comm = CComm.init_rank(uid, world, rank)
    layer = CAllGather(rows, cols, _spec(codec), comm=comm)
    fulls, digs = [], []
    import test_gpu_multiproc as M

    for x in M._inputs(rows, cols, seed=21):
        layer.step(torch.from_numpy(x[layer.lo:layer.hi]).cuda().to(torch.bfloat16))
        torch.cuda.synchronize()
        fulls.append(layer.reconstruction().cpu().numpy())
        digs.append(layer.digest())
    np.save(os.path.join(out_dir, f"f{rank}.npy"), np.stack(fulls))
    open(os.path.join(out_dir, f"d{rank}"), "wb").write(b"".join(digs))
    layer.close()
    comm.destroy()


@pytest.mark.parametrize("codec", ["quant2bit", "topk"])
def test_c_allgather_two_gpus_vs_reference_mesh(codec):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL cannot put two ranks on one device)")
    from paper_2507_17511_b200.comm import CComm

    import test_gpu_multiproc as M

    world, rows, cols = 2, 69, 3072
    uid = CComm.unique_id()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), uid, rows, cols, codec, d), nprocs=world, join=True)
        fulls = [np.load(os.path.join(d, f"f{r}.npy")) for r in range(world)]
        digs = [open(os.path.join(d, f"d{r}"), "rb").read() for r in range(world)]
    assert digs[0] == digs[1]
    ref = M._simulate_mesh(world, rows, cols, codec, "residual_with_feedback", seed=21)
    for f in fulls:
        assert f.tobytes() == ref.tobytes()
