"""Scale-mode cfg5: periodic 3D Taylor-Green projection steps on ONE B200
(BoxProjectionStepper).  usage: python tools/box_tgv.py p n steps"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_03032_b200 import geometry, timeint  # noqa: E402

p, n, steps = (int(a) for a in sys.argv[1:4])
import threading  # noqa: E402

_peak = [0]
_stop = threading.Event()


def _sample():  # device-wide memory in use (the C library allocates outside torch)
    while not _stop.is_set():
        free, total = torch.cuda.mem_get_info()
        _peak[0] = max(_peak[0], total - free)
        time.sleep(0.02)


torch.cuda.init()
_th = threading.Thread(target=_sample, daemon=True)
_th.start()
m = geometry.cartesian_mesh((n, n, n), lows=(-np.pi,) * 3, highs=(np.pi,) * 3,
                            periodic=(True,) * 3)
t0 = time.perf_counter()
st = timeint.BoxProjectionStepper(m, p, k=3, dt=0.02, nu=1.0 / 1600.0)


def tgv_u(x):
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    return np.stack([np.sin(X) * np.cos(Y) * np.cos(Z), -np.cos(X) * np.sin(Y) * np.cos(Z),
                     np.zeros_like(X)], axis=1)


st.initialize(st.vspace.project(tgv_u))
for _ in range(3):
    st.step()
torch.cuda.synchronize()
setup = time.perf_counter() - t0
its = []
t0 = time.perf_counter()
for _ in range(steps):
    r = st.step()
    its.append([r.mass_iters, r.pressure_iters, r.helmholtz_iters])
torch.cuda.synchronize()
ms = 1e3 * (time.perf_counter() - t0) / steps
st.profile = True
ph = st.step().phase_ms
_stop.set()
_th.join()
print(json.dumps({"p": p, "cells": n, "velocity_dofs": int(st.vspace.ndofs),
                  "pressure_dofs": int(st.pspace.ndofs), "ms_per_step": round(ms, 2),
                  "iterations_mass_pressure_helmholtz": its, "phase_ms": ph,
                  "setup_s": round(setup, 2), "kinetic_energy": st.kinetic_energy(),
                  "torch_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                  "device_peak_gb": round(_peak[0] / 1e9, 2),
                  "device_now_gb": round((lambda fi: fi[1] - fi[0])(torch.cuda.mem_get_info()) / 1e9, 2)}))
