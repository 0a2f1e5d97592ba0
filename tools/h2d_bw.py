import torch, time
for mb in (1, 8.65, 64, 512):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"H2D {mb} MB: best {ts[0]:.3f} ms ({n/ts[0]/1e6:.1f} GB/s) median {ts[5]:.3f} ms")
    ts = []
    for _ in range(10):
        e0.record(); h.copy_(d, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"D2H {mb} MB: best {ts[0]:.3f} ms ({n/ts[0]/1e6:.1f} GB/s) median {ts[5]:.3f} ms")

# freshly written source (the library writes its packed arrays right before the copy)
import numpy as np
for mb in (1, 8.65, 64):
    n = int(mb * 1e6)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    a = h.numpy()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for k in range(10):
        a[:] = k  # dirty every line in the CPU caches
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"H2D after host write {mb} MB: best {ts[0]:.3f} ms ({n/ts[0]/1e6:.1f} GB/s) median {ts[5]:.3f} ms")
    ts = []
    for k in range(10):
        a[:] = k
        t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); ts.append(1000*(time.perf_counter()-t0))
    ts.sort()
    print(f"  wall incl. launch: best {ts[0]:.3f} ms median {ts[5]:.3f} ms")

# several different pinned sources in turn (the library's per-plan uploads come from many buffers)
for nb, mb in ((8, 8.65), (32, 8.65)):
    n = int(mb * 1e6)
    hs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(nb)]
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    ts = []
    for k in range(3 * nb):
        e0.record(); d.copy_(hs[k % nb], non_blocking=True); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    ts = sorted(ts[nb:])
    print(f"H2D rotating over {nb} x {mb} MB: best {ts[0]:.3f} median {ts[len(ts)//2]:.3f} max {ts[-1]:.3f} ms")
