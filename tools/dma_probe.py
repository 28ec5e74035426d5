import torch, time, numpy as np, threading
n = 128 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print("pinned H2D GB/s", 10 * n / (time.perf_counter() - t) / 1e9)
src = np.ones(n, dtype=np.uint8)
dst = h.numpy()
for nt in (1, 4, 8, 16):
    t = time.perf_counter()
    for _ in range(5):
        ths = [threading.Thread(target=lambda i=i: np.copyto(dst[i*n//nt:(i+1)*n//nt], src[i*n//nt:(i+1)*n//nt])) for i in range(nt)]
        [x.start() for x in ths]; [x.join() for x in ths]
    print("host memcpy threads", nt, "GB/s", 5 * n / (time.perf_counter() - t) / 1e9)
