import ctypes, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1203_4031_b200.device import get_device
dev = get_device(); P = ctypes.c_void_p
for count in (1, 8):
    n = 4096
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.standard_normal((n, n)) / np.sqrt(n)).cuda()
    zs = [complex(0.1*np.cos(t), 0.05*np.sin(t)) for t in np.linspace(0.2, 2.9, count)]
    zr = (ctypes.c_double*count)(*[z.real for z in zs]); zi = (ctypes.c_double*count)(*[z.imag for z in zs])
    lu = torch.empty((2, count, n, n), dtype=torch.float64, device='cuda')
    piv = torch.empty((count, n), dtype=torch.int32, device='cuda')
    dd = int(dev.lib.fb_zgetrf_dinv_doubles(n))
    dinv = torch.empty((count, dd), dtype=torch.float64, device='cuda')
    info = torch.empty(count, dtype=torch.int32, device='cuda')
    buf = (ctypes.c_ulonglong*4)()
    dev.lib.fb_debug_panel_wall(buf)
    for rep in range(2):
        dev.lib.fb_debug_panel_wall(buf)
        dev.lib.fb_dense_shift_batched(dev.h, count, n, zr, zi, P(a.data_ptr()), None, n, None, None, n, P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n*n)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.lib.fb_zgetrf_batched(dev.h, count, n, P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n*n, P(piv.data_ptr()), n, P(dinv.data_ptr()), dd, P(info.data_ptr()))
        e1.record(); torch.cuda.synchronize()
        dev.lib.fb_debug_panel_wall(buf)
        ns, cyc, cnt = buf[0], buf[1], buf[2]
        print(f"sum of per-panel all-CTA spans {buf[3]/1e6:.2f} ms; count={count} LU {e0.elapsed_time(e1):.2f} ms; cluster panels (CTA0 of item 0..): {cnt} launches-CTAs, avg wall {ns/max(cnt,1)/1e3:.1f} us, avg {cyc/max(cnt,1):.0f} cycles -> {cyc/max(ns,1):.3f} GHz")

if os.environ.get("FB_PANEL_EVENTS"):
    cnt = ctypes.c_int(0)
    dev.lib.fb_debug_panel_events.restype = ctypes.c_double
    ms = dev.lib.fb_debug_panel_events(ctypes.byref(cnt))
    print(f"event-timed panel launches (all reps/items): {cnt.value}, avg {1e3 * ms / max(cnt.value, 1):.1f} us")
