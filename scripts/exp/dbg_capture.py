import torch, traceback
from paper_2507_17511_b200 import compressors as cx, comm, _lib
lib=_lib.load()
spec=cx.CompressorSpec(cx.CompressorKind("quant2bit"))
exs=[comm.PatchParallelExchange(4096,3072,spec) for _ in range(3)]
for e in exs[1:]: e.streams=exs[0].streams
x=torch.randn(4096,3072,device="cuda").to(torch.bfloat16)
for t in range(3):
    for e in exs: e.step(x)
    exs[-1].flush_decode()
torch.cuda.synchronize()
g=torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        for i,e in enumerate(exs):
            e.step(x); print("step",i,"ok", lib.cc_last_error(), torch.cuda.current_stream(), flush=True)
            st = torch.cuda.current_stream()
            print(" capture status", torch._C._cuda_isCurrentStreamCapturing(), flush=True)
        exs[-1].flush_decode()
        torch.cuda.current_stream().wait_stream(exs[0].streams.decode)
except Exception as ex:
    traceback.print_exc(); print("last err", lib.cc_last_error())
