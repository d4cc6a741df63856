"""Fused-step tile order sweep (gl_context_set_tile_order): kernel ms per
step for row-major vs vertical strips of n tiles, interleaved passes so clock
drift under the power cap hits every variant alike; the tensor hash after the
same steps must be identical for every order (bit-exactness).

usage: python tools/order_probe.py W H C steps order [order ...]
order = strip[:stack] (gl_context_set_tile_order); SM clocks are sampled
with nvidia-smi during each timed pass.
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_00572_b200 as g  # noqa: E402
from paper_1910_00572_b200.floorplan import make_floorplan, write_pgm  # noqa: E402
from bench import ClockSampler  # noqa: E402


def main():
    W, H, C, steps = (int(x) for x in sys.argv[1:5])
    orders = sys.argv[5:] or ["0", "8"]
    passes = int(os.environ.get("PASSES", "2"))
    ctx = g.Context(0)
    m = g.load_map(write_pgm(make_floorplan(W, H, seed=0)), 250, 0.1, ctx=ctx)
    ks = g.build_kernels(g.MotionNoise(), C, 0.1, 2 * math.pi / C)
    act = g.make_activation(m, ks, C, ctx)
    u = g.OdometryDelta(0.1, 0.0, 0.0)
    res = {o: [] for o in orders}
    hashes = {}
    t = None
    for p in range(passes):
        for o in orders:
            st, _, sk = o.partition(":")
            ctx.set_tile_order(int(st), int(sk or 0))
            clk = ClockSampler(0)
            clk.start()
            del t
            t = g.init_uniform(m, C, ctx)
            for _ in range(3):
                g.step_async(t, u, m, ks, act, ctx)
            ctx.synchronize()
            ctx.time_steps(True)
            ctx.mark(0)
            for _ in range(steps):
                g.step_async(t, u, m, ks, act, ctx)
            ctx.mark(1)
            ms = ctx.marks_ms(0, 1) / steps
            kms, kn = ctx.step_times()
            ctx.time_steps(False)
            g.tensor_status(t)
            c = clk.stop() or {}
            h = t.hash()
            hashes.setdefault(o, h)
            assert hashes[o] == h
            res[o].append((ms, kms / max(kn, 1), c.get("sm_mhz"), c.get("reasons")))
            time.sleep(0.5)
    ref = hashes[orders[0]]
    for o in orders:
        best = min(r[1] for r in res[o])
        print(f"{W}x{H}x{C} order={o:>5s} kern_ms best {best:.4f} all {[round(r[1], 4) for r in res[o]]} "
              f"step_ms {[round(r[0], 4) for r in res[o]]} sm_mhz {[r[2] for r in res[o]]} "
              f"{sorted(set(x for r in res[o] for x in (r[3] or [])))} hash_equal={hashes[o] == ref}", flush=True)


if __name__ == "__main__":
    main()
