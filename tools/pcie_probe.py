import torch, time
for n in (1e5, 1e6, 1e7):
    n = int(n)
    d = torch.randn(n, device="cuda")
    h = torch.empty(n).pin_memory()
    for rep in range(3):
        torch.cuda.synchronize()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record(); h.copy_(d, non_blocking=True); en.record(); torch.cuda.synchronize()
        t_d2h = st.elapsed_time(en)
        st.record(); d.copy_(h, non_blocking=True); en.record(); torch.cuda.synchronize()
        t_h2d = st.elapsed_time(en)
    print(f"{n*4/1e6:.1f} MB  D2H {t_d2h*1e3:.1f} us ({n*4/t_d2h/1e6:.1f} GB/s)  H2D {t_h2d*1e3:.1f} us ({n*4/t_h2d/1e6:.1f} GB/s)")
