import torch, time
n = 48 << 20
K = 16
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
def chunked(with_d2h, with_hbm):
    cur = torch.cuda.current_stream()
    for s in (s1, s2, s3): s.wait_stream(cur)
    c = n // K
    with torch.cuda.stream(s1):
        for i in range(K): d_a[i*c:(i+1)*c].copy_(h_in[i*c:(i+1)*c], non_blocking=True)
    if with_d2h:
        with torch.cuda.stream(s2):
            for i in range(K): h_out[i*c:(i+1)*c].copy_(d_b[i*c:(i+1)*c], non_blocking=True)
    if with_hbm:
        with torch.cuda.stream(s3):
            for i in range(6): big[: 1 << 29].copy_(big[1 << 29:])
    for s in (s1, s2, s3): cur.wait_stream(s)
print("H2D chunked alone %.3f ms" % t(lambda: chunked(False, False)))
print("H2D+D2H chunked %.3f ms" % t(lambda: chunked(True, False)))
print("H2D chunked + HBM copy %.3f ms" % t(lambda: chunked(False, True)))
print("H2D+D2H chunked + HBM copy %.3f ms" % t(lambda: chunked(True, True)))
print("HBM copy alone %.3f ms" % t(lambda: [big[: 1 << 29].copy_(big[1 << 29:]) for _ in range(6)]))
