import torch, time
n = 25165824 // 4
a = torch.empty(n, dtype=torch.float32, pin_memory=True); b = torch.empty(n, dtype=torch.float32, pin_memory=True)
da = torch.empty(n, device='cuda'); db = torch.empty(n, device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for _ in range(3):
    da.copy_(a, non_blocking=True); b.copy_(db, non_blocking=True)
torch.cuda.synchronize()
def t(f, k=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
print("h2d only ms", t(lambda: da.copy_(a, non_blocking=True)))
print("d2h only ms", t(lambda: b.copy_(db, non_blocking=True)))
def both():
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
print("both concurrent ms", t(both))
