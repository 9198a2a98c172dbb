"""D2H bandwidth into separately allocated pinned host buffers (placement variance probe)."""
import time
import torch

src = torch.empty(1 << 28, dtype=torch.float32, device="cuda")  # 1 GiB
for i in range(8):
    dst = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"buffer {i}: {4 * (1 << 28) / dt / 1e9:.1f} GB/s d2h", flush=True)
    keep = globals().setdefault("keep", [])
    keep.append(dst)
