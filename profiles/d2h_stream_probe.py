import torch, time
dev = torch.device('cuda', 0)
N = 2 << 30
src = torch.empty(N, dtype=torch.uint8, device=dev)
dst = torch.empty(N, dtype=torch.uint8).pin_memory()
s1, s2, s3, s4 = [torch.cuda.Stream() for _ in range(4)]
def one():
    dst.copy_(src, non_blocking=True)
def split(k, streams):
    h = N // k
    for i in range(k):
        with torch.cuda.stream(streams[i % len(streams)]):
            dst[i*h:(i+1)*h].copy_(src[i*h:(i+1)*h], non_blocking=True)
for name, fn in (("1 stream", one), ("2 streams", lambda: split(2, [s1, s2])), ("4 streams", lambda: split(4, [s1, s2, s3, s4]))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(name, N / dt / 1e9, "GB/s")
