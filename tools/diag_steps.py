"""Per-chunk step timing and belief max over a long c2 run (diagnostics)."""
import math
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1910_00572_b200 as g  # noqa: E402

W = H = 1024
C = 72
ctx = g.Context(0)
m = g.load_map(bench.make_map_bytes(W, H), 250, 0.1, ctx=ctx)
ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
act = g.make_activation(m, ks, C, ctx)
t = g.init_uniform(m, C, ctx)
u = g.OdometryDelta(0.1, 0.0, 0.0)
for chunk in range(12):
    ctx.synchronize()
    ctx.mark(0)
    for _ in range(100):
        g.step_async(t, u, m, ks, act, ctx)
    ctx.mark(1)
    ms = ctx.marks_ms(0, 1)
    import ctypes as Cc
    cnt = (Cc.c_uint64 * 4)()
    if hasattr(ctx.lib, "gl_debug_counters"):
        ctx.lib.gl_debug_counters(ctx.h, cnt)
    e = g.argmax_state(t)
    print(f"steps {100 * chunk:5d}-{100 * chunk + 99}: {ms / 100:.4f} ms/step  max {t.at(e.i, e.j, e.k):.3e}  exact epilogues so far {cnt[0]}", flush=True)
