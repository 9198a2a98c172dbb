"""fp32 dW = g^T A at the C2 trainer's layer shapes: one torch.mm against split-K
(strided-batched GEMM over P row chunks, then a sum of the P partials)."""
import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


for rows, hid, cols in [(169984, 256, 201), (16384, 256, 513)]:
    g = torch.randn(rows, hid, device=dev)
    A = torch.randn(rows, cols, device=dev)
    out = torch.empty(hid, cols, device=dev)
    ref = torch.mm(g.double().t(), A.double())
    base = t(lambda: torch.mm(g.t(), A, out=out))
    fl = 2 * rows * hid * cols
    print(f"rows {rows} hid {hid} cols {cols}: mm {base * 1e3:.0f} us ({fl / base / 1e9:.1f} TF/s)")
    for P in (4, 8, 16, 32, 64):
        ch = rows // P
        part = torch.empty(P, hid, cols, device=dev)

        def f():
            gv = g.as_strided((P, ch, hid), (ch * hid, hid, 1))
            av = A.as_strided((P, ch, cols), (ch * cols, cols, 1))
            torch.bmm(gv.transpose(1, 2), av, out=part)
            torch.sum(part, 0, out=out)
            if P * ch < rows:
                out.addmm_(g[P * ch:].t(), A[P * ch:])
        ms = t(f)
        err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
        print(f"  split-K P={P}: {ms * 1e3:.0f} us ({fl / ms / 1e9:.1f} TF/s)  max rel err {err:.2e}")
    for a_, b_ in [("gT A", lambda: torch.mm(g.t(), A, out=out)), ("(A^T g)^T", lambda: torch.mm(A.t(), g).t())]:
        print(f"  {a_}: {t(b_) * 1e3:.0f} us")

print("bf16 operands, fp32 output")
for rows, hid, cols in [(169984, 256, 201), (16384, 256, 513)]:
    g = torch.randn(rows, hid, device=dev).bfloat16()
    A = torch.randn(rows, cols, device=dev).bfloat16()
    out = torch.empty(hid, cols, device=dev)
    base = t(lambda: torch.mm(g.t(), A, out_dtype=torch.float32, out=out))
    print(f"rows {rows}: mm out_dtype fp32 {base * 1e3:.0f} us")
    for P in (4, 8, 16, 32):
        ch = rows // P
        part = torch.empty(P, hid, cols, device=dev)

        def f():
            gv = g.as_strided((P, ch, hid), (ch * hid, hid, 1))
            av = A.as_strided((P, ch, cols), (ch * cols, cols, 1))
            try:
                torch.bmm(gv.transpose(1, 2), av, out_dtype=torch.float32, out=part)
            except (RuntimeError, TypeError) as e:
                print("bmm out_dtype unsupported:", str(e)[:100])
                raise SystemExit
            torch.sum(part, 0, out=out)
        print(f"  split-K P={P}: {t(f) * 1e3:.0f} us")
