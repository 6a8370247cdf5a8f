import torch, time
n = 1445892
dev = torch.device("cuda")
h = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(5)]
d = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(5)]
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
def run(kind, reps=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps):
        if kind in ("h2d", "both"):
            with torch.cuda.stream(s_in):
                for i in range(3): d[i].copy_(h[i], non_blocking=True)
        if kind in ("d2h", "both"):
            with torch.cuda.stream(s_out):
                for i in range(3, 5): h[i].copy_(d[i], non_blocking=True)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
for k in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    t = run(k)
    print(k, f"{t*1e3:.3f} ms/step", "h2d GB/s" if k != "d2h" else "", f"{3*8*n/t/1e9:.1f}" if k != "d2h" else "", "d2h GB/s" if k != "h2d" else "", f"{2*8*n/t/1e9:.1f}" if k != "h2d" else "")
