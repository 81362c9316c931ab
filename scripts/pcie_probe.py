"""Pinned-host PCIe ceilings: H2D alone, D2H alone, both at once (256 MB each)."""
import torch
n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d(); d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms  {n / ms / 1e6:.1f} GB/s per direction", flush=True)

# chunked pipeline without compute: H2D of chunk c on s1, D2H of chunk c on s2 after it
for nch in (4, 16, 32, 128):
    cs = n // nch
    evs = [torch.cuda.Event() for _ in range(nch)]

    def piped():
        for c in range(nch):
            with torch.cuda.stream(s1):
                d1[c * cs:(c + 1) * cs].copy_(h1[c * cs:(c + 1) * cs], non_blocking=True)
                evs[c].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(evs[c])
                h2[c * cs:(c + 1) * cs].copy_(d2[c * cs:(c + 1) * cs], non_blocking=True)
    ms = t(piped)
    print(f"piped {nch} chunks: {ms:.2f} ms", flush=True)

# copies while kernels run on a third stream
import sys as _s, os as _o  # noqa: E402
_s.path.insert(0, _o.path.dirname(_o.path.dirname(_o.path.abspath(__file__))))
import paper_1406_1717_b200 as mf  # noqa: E402
xs = mf.generate_device("uniform_f32", 2, 1 << 26)
ys = torch.empty_like(xs)
s3 = torch.cuda.Stream()
for kk in (3, 1023):
    def busy():
        with torch.cuda.stream(s3):
            for _ in range(3):
                mf.median_filter_device(xs, kk, out=ys)
    busy(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s3); busy(); b.record(s3); torch.cuda.synchronize()
    kms = a.elapsed_time(b)
    a2, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a3, b3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a3.record(s3); busy(); b3.record(s3)
    a2.record(s1); h2d(); b2.record(s1)
    torch.cuda.synchronize()
    print(f"k={kk}: kernels alone {kms:.2f} ms, with h2d {a3.elapsed_time(b3):.2f} ms; h2d alongside {a2.elapsed_time(b2):.2f} ms", flush=True)
