import time, os, numpy as np, threading, torch
n = 1 << 28  # 2 GiB of u64
a = np.ones(n, dtype=np.uint64); b = np.empty_like(a)
for _ in range(2): np.copyto(b, a)
t=time.perf_counter(); np.copyto(b, a); dt=time.perf_counter()-t
print(f"numpy single-thread copy: {2*a.nbytes/dt/1e9:.1f} GB/s (read+write)")
T = os.cpu_count()
def part(i):
    lo, hi = n*i//T, n*(i+1)//T
    np.copyto(b[lo:hi], a[lo:hi])
for _ in range(2):
    ths=[threading.Thread(target=part, args=(i,)) for i in range(T)]
    t=time.perf_counter(); [x.start() for x in ths]; [x.join() for x in ths]; dt=time.perf_counter()-t
print(f"numpy {T}-thread copy: {2*a.nbytes/dt/1e9:.1f} GB/s (read+write)")
def rd(i):
    lo, hi = n*i//T, n*(i+1)//T
    a[lo:hi].sum()
for _ in range(2):
    ths=[threading.Thread(target=rd, args=(i,)) for i in range(T)]
    t=time.perf_counter(); [x.start() for x in ths]; [x.join() for x in ths]; dt=time.perf_counter()-t
print(f"numpy {T}-thread read (sum): {a.nbytes/dt/1e9:.1f} GB/s")
h = torch.empty(n, dtype=torch.int64, pin_memory=True); d = torch.empty(n, dtype=torch.int64, device='cuda')
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize(); t=time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); dt=time.perf_counter()-t
print(f"pinned H2D: {h.numel()*8/dt/1e9:.1f} GB/s")
print("cpus", os.cpu_count(), open('/proc/cpuinfo').read().count('processor'))
