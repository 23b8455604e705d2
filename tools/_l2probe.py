"""Probe: does a persisting access-policy window keep a buffer in L2 across a 256 MiB flush?"""
import torch
from cuda.bindings import runtime as r

torch.cuda.init()
dev = 0
_, maxp = r.cudaDeviceGetAttribute(r.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, dev)
print("max persisting", maxp, r.cudaDeviceSetLimit(r.cudaLimit.cudaLimitPersistingL2CacheSize, 32 << 20))
buf = torch.ones(8 << 20, dtype=torch.float32, device="cuda")  # 32 MiB
junk = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()


def t_read(n=20, flush=True):
    ts = []
    for _ in range(n):
        if flush:
            junk.fill_(1.0)
        torch.cuda._sleep(100_000)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); buf.sum(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


print("warm   ", t_read(flush=False))
print("flushed", t_read())
attr = r.cudaStreamAttrValue()
w = attr.accessPolicyWindow
w.base_ptr = buf.data_ptr(); w.num_bytes = buf.numel() * 4; w.hitRatio = 1.0
w.hitProp = r.cudaAccessProperty.cudaAccessPropertyPersisting
w.missProp = r.cudaAccessProperty.cudaAccessPropertyStreaming
attr.accessPolicyWindow = w
print(r.cudaStreamSetAttribute(s.cuda_stream, r.cudaStreamAttrID.cudaLaunchAttributeAccessPolicyWindow, attr))
for _ in range(3):
    buf.sum()
print("pinned warm   ", t_read(flush=False))
print("pinned flushed", t_read())
