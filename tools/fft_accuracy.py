"""FFT accuracy probe: the device transform (tsf_fft_debug) vs an exact
long-double DFT (scipy.fft in long double), beside numpy pocketfft's own
error.  Usage: python tools/fft_accuracy.py [N ...]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import scipy.fft as sf
import torch

from paper_2002_11978_b200 import _native

lib = _native.load()
rng = np.random.default_rng(11)
for N in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
    B = 64
    x = rng.standard_normal((B, N)) + 1j * rng.standard_normal((B, N))
    xr = rng.standard_normal((B, N)) + 0j
    for name, data in (("complex", x), ("real", xr)):
        for inv in (0, 1):
            d_in = torch.from_numpy(data.astype(np.complex128)).cuda()
            d_out = torch.empty_like(d_in)
            _native.check(lib.tsf_fft_debug(N, inv, B, d_in.data_ptr(), d_out.data_ptr(),
                                            _native.stream_ptr()))
            got = d_out.cpu().numpy()
            dl = data.astype(np.clongdouble)
            ex = sf.ifft(dl, axis=1) * N if inv else sf.fft(dl, axis=1)
            ref = np.fft.ifft(data, axis=1) * N if inv else np.fft.fft(data, axis=1)
            rel = lambda a: float(np.linalg.norm((a.astype(np.clongdouble) - ex)) /
                                  np.linalg.norm(ex))
            print(f"N={N} {name:7s} {'inv' if inv else 'fwd'}: device {rel(got):.3e} "
                  f"numpy {rel(ref):.3e}", flush=True)
