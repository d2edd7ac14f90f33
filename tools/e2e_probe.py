import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1803_06058_b200 import LoveCache
from synth import get_config, make_inputs
p = get_config(2); inp = make_inputs(p)
kw = dict(m=p.m, lo=p.lo, h=p.h, lengthscale=p.lengthscale, outputscale=p.outputscale, sigma2=p.sigma2, k=p.k, precision=p.precision)
Xh = torch.from_numpy(inp.X).pin_memory(); yh = torch.from_numpy(inp.y).pin_memory(); Xsh = torch.from_numpy(inp.Xs).pin_memory()
s = torch.cuda.current_stream()
def ev(): return torch.cuda.Event(enable_timing=True)
for it in range(4):
    e = [ev() for _ in range(8)]
    e[0].record(s)
    X = Xh.to('cuda', non_blocking=True); y = yh.to('cuda', non_blocking=True); e[1].record(s)
    c = LoveCache.build(X, y, **kw); e[2].record(s)
    Xs = Xsh.to('cuda', non_blocking=True); e[3].record(s)
    v = c.predict_var(Xs); e[4].record(s)
    t0 = time.perf_counter(); vh = v.cpu(); t1 = time.perf_counter(); e[5].record(s)
    out = torch.empty(v.shape, dtype=v.dtype, pin_memory=True); out.copy_(v, non_blocking=True); e[6].record(s)
    c.free(); e[7].record(s)
    e[7].synchronize()
    names = ['h2d X,y', 'build', 'h2d Xs', 'predict', 'd2h pageable', 'd2h pinned', 'free']
    print(' '.join('%s %.3f' % (n, e[i].elapsed_time(e[i+1])) for i, n in enumerate(names)), 'cpu(.cpu()) %.3f ms' % ((t1-t0)*1e3))
# also: build directly from the host tensors (what the bench e2e does)
for it in range(3):
    a, b = ev(), ev(); a.record(s)
    c = LoveCache.build(Xh, yh, **kw); v = c.predict_var(Xsh); vh = v.cpu(); c.free()
    b.record(s); b.synchronize(); print('bench-style e2e step %.3f ms' % a.elapsed_time(b))
