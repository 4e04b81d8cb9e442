"""The exchanges over REAL NCCL collectives, one process per GPU (needs >= 2 GPUs;
skipped on 1-GPU boxes, where tests/test_gpu_multiproc.py runs the same checks
with every rank on cuda:0 over gloo).  Same oracle comparison: every rank's
reconstruction equals the reference mesh simulation bit for bit after every
step, and all ranks' digests agree (mesh.py:188-237, 320-324)."""

import pytest
import torch

import test_gpu_multiproc as M

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpus():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")


def _world(w):
    if torch.cuda.device_count() < w:
        pytest.skip(f"needs {w} GPUs")
    return w


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("codec", ["quant2bit", "sign1bit", "topk"])
def test_patch_allgather_nccl(world, codec):
    M._run_patch(_world(world), 32 * world + 5, 3072, codec, backend="nccl")


@pytest.mark.parametrize("world", [2, 4])
def test_ring_nccl(world):
    M._run_patch(_world(world), 16 * world + 3, 3072, "quant2bit", topology="ring", backend="nccl")


@pytest.mark.parametrize("world", [2, 8])
def test_ulysses_nccl(world):
    M._run_ulysses(_world(world), 3072, "sign1bit", backend="nccl")
