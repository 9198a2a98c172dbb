import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2305_16588_b200 import _lib
lib = _lib.lib()
for n in [1 << 20, 111_000_000]:
    tot = torch.from_numpy((np.random.default_rng(1).zipf(1.3, n) % (1 << 40)).astype(np.int64)).cuda()
    tot[::7] = 0
    out = torch.empty(n, dtype=torch.int64, device='cuda')
    tmp = torch.empty(lib.gc_descending_order_temp_bytes(n), dtype=torch.uint8, device='cuda')
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _lib.check(lib.gc_descending_order(tot.data_ptr(), n, out.data_ptr(), tmp.data_ptr(), tmp.numel(), _lib.stream_handle()))
        torch.cuda.synchronize(); t1 = time.perf_counter()
    want = torch.from_numpy(np.lexsort((np.arange(n), -tot.cpu().numpy()))).cuda()
    print(n, f"{(t1-t0)*1e3:.2f} ms", bool(torch.equal(out, want)))
    s = torch.empty(n, dtype=torch.int64, device='cuda')
    stmp = torch.empty(lib.gc_order_scan_temp_bytes(n), dtype=torch.uint8, device='cuda')
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _lib.check(lib.gc_hot_prefix(tot.data_ptr(), out.data_ptr(), n, s.data_ptr(), stmp.data_ptr(), stmp.numel(), _lib.stream_handle()))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print("hot_prefix", f"{(t1-t0)*1e3:.2f} ms", bool(torch.equal(s, torch.cumsum(tot[out], 0))))
