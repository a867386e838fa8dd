"""HBM bandwidth for read/write mixes (torch element-wise ops on 4 GiB fields; best of 5, CUDA events).
Context for the x pass, whose mix is 4 reads : 3 writes."""
import torch

n = 1 << 30  # float32 elements = 4 GiB per field
a, b, c, d = (torch.rand(n, device="cuda") for _ in range(4))
torch.cuda.synchronize()


def t(fn, nbytes):
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{fn.__name__:10s} {nbytes / best / 1e6:8.1f} GB/s ({best:.2f} ms)")


def read_only(): torch.sum(a)
def write_only(): d.fill_(1.0)
def copy_1r1w(): d.copy_(a)
def add_2r1w(): torch.add(a, b, out=d)
def addcmul_3r1w(): torch.addcmul(a, b, c, out=d)
for fn, k in [(read_only, 1), (write_only, 1), (copy_1r1w, 2), (add_2r1w, 3), (addcmul_3r1w, 4)]:
    t(fn, 4 * n * k)
