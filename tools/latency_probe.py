import sys, time
sys.path.insert(0, '/root/repo')
import paper_2603_26576_b200 as hb
def mk(k):
    host = [hb.HostRecord(j % 4, hb.HostState.OFFLOAD if j % 3 == 1 else hb.HostState.USEFUL, hb.Interval(j * 10, j * 10 + 5)) for j in range(k)]
    dev = [hb.DeviceRecord(h.rank, hb.DeviceActivityKind.KERNEL, hb.Interval(h.interval.start + 1, h.interval.end), None) for h in host]
    return hb.Trace(host_processes=(0, 1, 2, 3), devices=tuple(hb.DeviceDecl(d, d) for d in range(4)), host_records=tuple(host), device_records=tuple(dev))
for k in (20, 1000, 100000):
    t = mk(k)
    for _ in range(5): hb.compute_report(t)
    n = 200 if k < 100000 else 20
    t0 = time.perf_counter()
    for _ in range(n): r = hb.compute_report(t)
    dt = (time.perf_counter() - t0) / n
    print(f"compute_report of {2*k} records: {dt*1e6:.0f} us per call")
