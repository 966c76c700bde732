import time, numpy as np, torch, json
cr = torch.cuda.cudart()
out={}
for gb in (0.26, 2.6):
    a = np.ones(int(gb*1e9)//2, np.uint16)
    for flag in (0, 2):  # default, mapped? (cudaHostRegisterMapped=2)
        t0=time.perf_counter(); r=cr.cudaHostRegister(a.ctypes.data, a.nbytes, flag); t1=time.perf_counter()
        cr.cudaHostUnregister(a.ctypes.data); t2=time.perf_counter()
        out[f"{gb}GB_flag{flag}"]=dict(register_ms=1e3*(t1-t0), unregister_ms=1e3*(t2-t1), rc=int(r))
print(json.dumps(out))
