"""PCIe copy pipelines of bench.py's e2e round trip, without the step: the C3 reference-layout
state (pos, vel, rho, vel_prev, rho_prev f32 + id i64: 52 B/row, 530 MB) moved in row chunks
of six copies each -- H2D alone, D2H alone, and the chained round trip (H2D of chunk c after
the D2H of chunk c), against one 530 MB copy per direction.
  python tools/pcie_chunks.py"""
import torch

n = 10_200_478
W = {"pos": 3, "vel": 3, "rho": 1, "vel_prev": 3, "rho_prev": 1}
h = {k: torch.empty((n, w) if w > 1 else (n,), dtype=torch.float32, pin_memory=True) for k, w in W.items()}
d = {k: torch.empty_like(v, device="cuda") for k, v in h.items()}
h["id"] = torch.empty(n, dtype=torch.int64, pin_memory=True)
d["id"] = torch.empty(n, dtype=torch.int64, device="cuda")
pairs = [(h[k], d[k]) for k in h]
nbytes = sum(x.numel() * x.element_size() for x, _ in pairs)
big_h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
big_d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def bounds(nch):
    return [(n * c // nch, n * (c + 1) // nch) for c in range(nch)]


def h2d(nch):
    def f():
        for lo, hi in bounds(nch):
            for hb, db in pairs:
                db[lo:hi].copy_(hb[lo:hi], non_blocking=True)
    return f


def d2h(nch):
    def f():
        for lo, hi in bounds(nch):
            for hb, db in pairs:
                hb[lo:hi].copy_(db[lo:hi], non_blocking=True)
    return f


def chained(nch):
    def f():
        cur = torch.cuda.current_stream()
        s_out.wait_stream(cur)
        evs = []
        with torch.cuda.stream(s_out):
            for lo, hi in bounds(nch):
                for hb, db in pairs:
                    hb[lo:hi].copy_(db[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_out)
                evs.append(e)
        with torch.cuda.stream(s_in):
            for (lo, hi), e in zip(bounds(nch), evs):
                s_in.wait_event(e)
                for hb, db in pairs:
                    db[lo:hi].copy_(hb[lo:hi], non_blocking=True)
        cur.wait_stream(s_in)
    return f


def both_chunked(nch):
    def f():
        cur = torch.cuda.current_stream()
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        with torch.cuda.stream(s_out):
            d2h(nch)()
        with torch.cuda.stream(s_in):
            h2d(nch)()
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
    return f


def chained_big(nch):
    """the same round trip on one contiguous buffer per direction (one copy per chunk)"""
    def f():
        cur = torch.cuda.current_stream()
        s_out.wait_stream(cur)
        evs = []
        b = [(nbytes * c // nch, nbytes * (c + 1) // nch) for c in range(nch)]
        with torch.cuda.stream(s_out):
            for lo, hi in b:
                big_h[lo:hi].copy_(big_d[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_out)
                evs.append(e)
        with torch.cuda.stream(s_in):
            for (lo, hi), e in zip(b, evs):
                s_in.wait_event(e)
                big_d[lo:hi].copy_(big_h[lo:hi], non_blocking=True)
        cur.wait_stream(s_in)
    return f


def both_big():
    cur = torch.cuda.current_stream()
    s_in.wait_stream(cur)
    s_out.wait_stream(cur)
    with torch.cuda.stream(s_in):
        big_d.copy_(big_h, non_blocking=True)
    with torch.cuda.stream(s_out):
        big_h.copy_(big_d, non_blocking=True)
    cur.wait_stream(s_in)
    cur.wait_stream(s_out)


gb = nbytes / 1e9
print(f"state {gb:.3f} GB per direction")
print(f"one copy: H2D {timed(lambda: big_d.copy_(big_h, non_blocking=True)):.2f} ms, "
      f"D2H {timed(lambda: big_h.copy_(big_d, non_blocking=True)):.2f} ms, both at once {timed(both_big):.2f} ms")
for nch in (1, 2, 4, 8, 16):
    print(f"{nch:2d} chunks x 6 arrays: H2D {timed(h2d(nch)):.2f} ms, D2H {timed(d2h(nch)):.2f} ms, "
          f"chained round trip {timed(chained(nch)):.2f} ms, both directions unchained "
          f"{timed(both_chunked(nch)):.2f} ms, chained on one contiguous buffer {timed(chained_big(nch)):.2f} ms")
