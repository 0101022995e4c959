"""Host<->device copy rates of 25 MiB pinned buffers: H2D alone, D2H alone, both at once (two streams)."""
import torch, time
n = 25 * 1024 * 1024
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
for nm, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn); print(nm, round(ms, 3), "ms", round(n / ms / 1e6, 1), "GB/s per direction")


# the bench's e2e pipeline shape: per step H2D of a 25 MiB input, a compute stage of C us on the main
# stream, D2H of a 25 MiB output; two buffers; per-step device time over K steps
def pipeline(K, compute_us, reuse_wait=True, nb=2):
    main = torch.cuda.current_stream()
    xs = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(nb)]
    ys = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(nb)]
    yh = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(nb)]
    spin = torch.empty(1 << 20, device="cuda")
    ev = lambda: torch.cuda.Event()  # noqa: E731
    eh, ec, ed = [ev() for _ in range(K)], [ev() for _ in range(K)], [ev() for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(main)
    s1.wait_event(t0)
    for i in range(K):
        bb = i % nb
        with torch.cuda.stream(s1):
            if i >= nb and reuse_wait:
                s1.wait_event(ec[i - nb])
            xs[bb].copy_(h1, non_blocking=True)
            eh[i].record(s1)
        main.wait_event(eh[i])
        if i >= nb and reuse_wait:
            main.wait_event(ed[i - nb])
        if compute_us:
            torch.cuda._sleep(int(compute_us * 1965))   # ~cycles at 1.965 GHz
        ys[bb].copy_(xs[bb])
        ec[i].record(main)
        with torch.cuda.stream(s2):
            s2.wait_event(ec[i])
            yh[bb].copy_(ys[bb], non_blocking=True)
            ed[i].record(s2)
    main.wait_event(ed[K - 1])
    t1.record(main)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / K


for nb in (2, 3, 4):
    for c in (0, 210):
        pipeline(6, c, nb=nb)
        print(f"pipeline buffers={nb} K=20 compute={c} us: {pipeline(20, c, nb=nb):.3f} ms/step")
