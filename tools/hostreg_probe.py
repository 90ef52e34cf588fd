"""Probe cudaHostRegister limits on POSIX shm regions (sizes, flags)."""
import ctypes, mmap, os
import torch
torch.cuda.init()
cudart = ctypes.CDLL("libcudart.so.12") if False else None
libc = ctypes.CDLL(None)
rt = torch.cuda.cudart()
for gb in (1, 4, 6, 12, 24):
    n = gb << 30
    name = f"/fcdp_probe_{gb}"
    fd = os.open(f"/dev/shm{name}", os.O_CREAT | os.O_RDWR, 0o600)
    os.ftruncate(fd, n)
    m = mmap.mmap(fd, n)
    buf = (ctypes.c_char * 1).from_buffer(m)
    ptr = ctypes.addressof(buf)
    for flags in (0, 1, 2, 3):  # Default, Portable, Mapped, Portable|Mapped
        err = rt.cudaHostRegister(ptr, n, flags)
        ok = int(err) if not isinstance(err, int) else err
        print(f"{gb} GiB flags={flags}: {err}", flush=True)
        if str(err).endswith("cudaSuccess") or ok == 0:
            rt.cudaHostUnregister(ptr)
    del buf
    m.close()
    os.close(fd)
    os.unlink(f"/dev/shm{name}")
