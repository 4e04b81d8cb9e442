"""Experiment: the receiver decode on a green-context stream confined to N SMs (SM
partition between the decode and K1), vs the plain decode stream.  Config-1 step
(57 layers, [4096, 3072] quant2bit loopback), graph replay when capturable, else eager.
python scripts/exp/green_ab.py <decode_sms> [k1_grid]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from cuda.bindings import driver as drv  # noqa: E402

import bench  # noqa: E402
from paper_2507_17511_b200 import comm  # noqa: E402
from paper_2507_17511_b200 import compressors as cx  # noqa: E402


def _ctx_stream(dev, res):
    err, desc = drv.cuDevResourceGenerateDesc([res], 1)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, g = drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    err, st = drv.cuGreenCtxStreamCreate(g, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    return torch.cuda.ExternalStream(int(st)), g


def green_stream(nsm, split_rest=False):
    """(decode stream on nsm SMs, [compute stream on the remaining SMs])"""
    torch.cuda.init()
    err, dev = drv.cuDeviceGet(0)
    err, res = drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM)
    err, groups, n, rem = drv.cuDevSmResourceSplitByCount(1, res, 0, nsm)
    assert err == drv.CUresult.CUDA_SUCCESS, err
    print("green ctx SMs", groups[0].sm.smCount, "rest", rem.sm.smCount, file=sys.stderr)
    out = [_ctx_stream(dev, groups[0])]
    if split_rest:
        out.append(_ctx_stream(dev, rem))
    return out


def main():
    nsm = int(sys.argv[1])
    L, rows, cols = 57, 4096, 3072
    dev = torch.device("cuda", 0)
    spec = cx.CompressorSpec(cx.CompressorKind.QUANT2BIT)
    split = len(sys.argv) > 2 and sys.argv[2] == "split"
    keep = None
    if nsm > 0:
        keep = green_stream(nsm, split)
        if split:
            torch.cuda.set_stream(keep[1][0])  # K1 (compute) on the complementary SMs
    exs = [comm.PatchParallelExchange(rows, cols, spec) for _ in range(L)]
    for e in exs[1:]:
        e.streams = exs[0].streams
    S = exs[0].streams
    if nsm > 0:
        S._decode = keep[0][0]
    inputs = [bench.flux_inputs(rows, cols, 0, rows, l, dev) for l in range(L)]

    def one(par):
        for l, e in enumerate(exs):
            e.step(inputs[l][par])

    one(0)
    for s in range(3):
        one((s + 1) % 2)
    torch.cuda.synchronize()
    mode = "eager"
    try:
        gr = []
        for p in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=S.compute if split else None):
                one(p)
                torch.cuda.current_stream().wait_stream(S.decode)
            gr.append(g)
        for e in exs:
            e.after_capture()
        mode = "graph"
    except Exception as exc:  # noqa: BLE001
        print("capture failed:", type(exc).__name__, str(exc)[:200], file=sys.stderr)
        torch.cuda.synchronize()
        gr = None
    K = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(S.compute)
    for k in range(K):
        if gr:
            gr[k % 2].replay()
        else:
            one(k % 2)
    S.compute.wait_stream(S.decode)
    b.record(S.compute)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    print({"decode_sms": nsm, "mode": mode, "us_per_layer": round(ms / L * 1e3, 2),
           "GBs": round(L * 2 * rows * cols / (ms / 1e3) / 1e9, 1)}, flush=True)
    del keep


if __name__ == "__main__":
    main()
