"""cProfile of the drop-in compute_report on a tiny trace (40 records): where the per-call
microseconds go outside the kernel.  python tools/api_profile.py"""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import paper_2603_26576_b200 as hb
def mk(k):
    host = [hb.HostRecord(j % 4, hb.HostState.OFFLOAD if j % 3 == 1 else hb.HostState.USEFUL, hb.Interval(j * 10, j * 10 + 5)) for j in range(k)]
    dev = [hb.DeviceRecord(h.rank, hb.DeviceActivityKind.KERNEL, hb.Interval(h.interval.start + 1, h.interval.end), None) for h in host]
    return hb.Trace(host_processes=(0, 1, 2, 3), devices=tuple(hb.DeviceDecl(d, d) for d in range(4)), host_records=tuple(host), device_records=tuple(dev))
t = mk(20)
for _ in range(50): hb.compute_report(t)
pr = cProfile.Profile()
pr.enable()
for _ in range(1000): hb.compute_report(t)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(25)
