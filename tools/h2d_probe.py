"""Host->device copy bandwidth from pinned memory (4 GiB of int32, one or two streams, whole or in
16 chunks): the floor of the host-buffer (e2e) path, which must move the label volume over PCIe.
usage: python tools/h2d_probe.py"""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    torch.cuda.synchronize(); t = time.perf_counter()
    half = n // 2
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t
    # 16 chunks on one stream
    torch.cuda.synchronize(); t = time.perf_counter()
    c = n // 16
    for i in range(16): d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter() - t
    # 16 chunks alternating 2 streams
    torch.cuda.synchronize(); t = time.perf_counter()
    for i in range(16):
        with torch.cuda.stream(s1 if i % 2 == 0 else s2): d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter() - t
    print(f"1 stream {4*n/t1/1e9:.1f} GB/s ({t1*1e3:.1f} ms); 2 streams {4*n/t2/1e9:.1f} GB/s; 16 chunks {4*n/t3/1e9:.1f}; 16 chunks/2 streams {4*n/t4/1e9:.1f}")
