import time, numpy as np, torch
cr = torch.cuda.cudart()
a = np.ones(537_000_000 // 4, np.float32); b = np.ones(134_000_000, np.uint8)
da = torch.empty(a.size, dtype=torch.float32, device='cuda'); db = torch.empty(b.size, dtype=torch.uint8, device='cuda')
for i in range(3):
    t0 = time.perf_counter()
    cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0); cr.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
    t1 = time.perf_counter()
    da.copy_(torch.from_numpy(a), non_blocking=True); db.copy_(torch.from_numpy(b), non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data); cr.cudaHostUnregister(b.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms  H2D {1e3*(t2-t1):.1f} ms ({(a.nbytes+b.nbytes)/(t2-t1)/1e9:.1f} GB/s)  unregister {1e3*(t3-t2):.1f} ms", flush=True)
