"""Experiment: does a degree-descending vertex layout speed up the lpa() loop?
Builds R-MAT on the device, relabels it with torch (positions sorted by degree desc,
ties by a hash of the id), wraps the relabelled arrays and times lpa() on both layouts."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2411_11468_b200 import labelprop as lp, _capi

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dg = lp.DeviceGraph.rmat(scale, 16, 1)
n, m2 = dg.n, dg.m2
c = dg.device_csr()
dev = torch.device("cuda:0")
off = torch.empty(n + 1, dtype=torch.int64, device=dev)
tgt = torch.empty(m2, dtype=torch.int32, device=dev)
cud = C.CDLL("libcudart.so") if False else None
# copy the resident arrays into torch tensors (device to device)
import cuda.bindings.runtime as rt  # cuda-python
rt.cudaMemcpy(off.data_ptr(), c.offsets, (n + 1) * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
rt.cudaMemcpy(tgt.data_ptr(), c.targets, m2 * 4, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
torch.cuda.synchronize()

def run(g, label):
    cfg = lp.LpaConfig()
    t = lp.Tuning(profile=True)
    for _ in range(3):
        g.lpa(cfg, t, want_host=False)
    rs = [g.lpa(cfg, t, want_host=False) for _ in range(3)]
    loop = sum(r.stats.elapsed_seconds for r in rs) / 3
    print(f"{label}: loop {loop*1e3:.1f} ms iters {rs[-1].stats.iterations} "
          f"edges/s {m2/loop/1e9:.2f}G dn {rs[-1].stats.delta_n_per_iter}", flush=True)

run(dg, "original")
t0 = time.time()
deg = (off[1:] - off[:-1])
ids = torch.arange(n, device=dev, dtype=torch.int64)
h = (ids * 0x9E3779B1) & 0xFFFFFFFF
h = h ^ (h >> 16)
key = ((deg.max() - deg) << 32) | h
perm = torch.argsort(key)
inv = torch.empty_like(perm)
inv[perm] = ids
ndeg = deg[perm]
noff = torch.zeros(n + 1, dtype=torch.int64, device=dev)
noff[1:] = torch.cumsum(ndeg, 0)
ntgt = torch.empty(m2, dtype=torch.int32, device=dev)
inv32 = inv.to(torch.int32)
CH = 1 << 27
p0 = 0
while p0 < n:
    # chunk of positions with <= CH edges (at least one vertex)
    p1 = int(torch.searchsorted(noff, noff[p0] + CH, right=True)) - 1
    p1 = max(p1, p0 + 1)
    p1 = min(p1, n)
    e0, e1 = int(noff[p0]), int(noff[p1])
    if e1 > e0:
        pe = torch.repeat_interleave(torch.arange(p0, p1, device=dev), ndeg[p0:p1])
        old = off[perm[pe]] + (torch.arange(e0, e1, device=dev) - noff[pe])
        ntgt[e0:e1] = inv32[tgt[old].long()]
        del pe, old
    p0 = p1
torch.cuda.synchronize()
print(f"relabel on device (torch): {time.time()-t0:.2f} s", flush=True)
del tgt
csr = _capi.nulpa_csr()
csr.n, csr.m2 = n, m2
csr.offsets, csr.targets, csr.weights = noff.data_ptr(), ntgt.data_ptr(), None
hdl = C.c_void_p()
dg.free()
_capi.check(_capi.lib().nulpa_graph_wrap_device(C.byref(csr), 0, C.byref(hdl)))
g2 = lp.DeviceGraph(hdl.value, 0)
run(g2, "degree-sorted")
cfg = lp.LpaConfig()
t = lp.Tuning(profile=True, schedule=1)
for _ in range(2):
    g2.lpa(cfg, t, want_host=False)
rs = [g2.lpa(cfg, t, want_host=False) for _ in range(3)]
loop = sum(r.stats.elapsed_seconds for r in rs) / 3
print(f"degree-sorted, ascending schedule: loop {loop*1e3:.1f} ms iters {rs[-1].stats.iterations}", flush=True)
