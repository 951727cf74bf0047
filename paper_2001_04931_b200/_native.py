"""ctypes binding of the C ABI in include/empc_b200.h.

The shared library ``libempc_b200.so`` (built in-tree by
``__graft_entry__.build()`` / ``make -C paper_2001_04931_b200/csrc``) is the
only compute path: there is no CPU fallback.  Importing this module never
touches the GPU; the library is loaded on first use and a missing library
raises immediately.
"""

from __future__ import annotations

import collections
import ctypes as C
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libempc_b200.so")

EMPC_OK, EMPC_EINVAL, EMPC_ECUDA, EMPC_ESTATE, EMPC_ENOMEM = 0, -1, -2, -3, -4
EMPC_FP32, EMPC_FP64 = 0, 1
EMPC_OPT_PERSISTENT, EMPC_OPT_HALF_K, EMPC_OPT_INCREMENTAL_SELECT, EMPC_OPT_RADIX_SELECT = 1, 2, 3, 4
EMPC_OPT_PERSIST_TILE, EMPC_OPT_SMALL_SOLVE = 5, 6

# every symbol include/empc_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "empc_create", "empc_destroy", "empc_last_error", "empc_set_schedule", "empc_set_scorer", "empc_set_problems",
    "empc_pop_alloc", "empc_pop_free", "empc_pop_read", "empc_pop_write", "empc_run", "empc_score",
    "empc_select", "empc_expand", "empc_time_device", "empc_describe", "empc_num_variants",
    "empc_set_variant", "empc_set_occupancy", "empc_set_tensor_cores", "empc_set_option", "empc_philox", "empc_shard_setup", "empc_shard_entry_bytes",
    "empc_shard_init", "empc_shard_export", "empc_shard_import", "empc_shard_evolve", "empc_shard_read", "empc_get_stream",
    "empc_plant_linearize_discretize", "empc_plant_integrate", "empc_plant_last_error",
)

EMPC_PLANT_PENDULUM, EMPC_PLANT_NLINK = 0, 1
EMPC_DISCRETIZE_EXACT, EMPC_DISCRETIZE_EULER = 0, 1


class empc_dims(C.Structure):
    _fields_ = [(f, C.c_int32) for f in
                ("n", "m", "T", "p", "num_sims", "num_parents", "instances", "dense_q", "precision", "device")]


class empc_injected(C.Structure):
    _fields_ = [
        ("init", C.c_void_p),
        ("parents", C.c_void_p),
        ("take_second", C.c_void_p),
        ("mutate", C.c_void_p),
        ("noise", C.c_void_p),
    ]


class empc_run_args(C.Structure):
    _fields_ = [
        ("init", C.c_int32),
        ("rescore", C.c_int32),
        ("evolves", C.c_int32),
        ("slot_in", C.c_int32),
        ("slot_out", C.c_int32),
        ("generation0", C.c_int64),
        ("seed", C.c_uint64),
        ("mutation_prob", C.c_double),
        ("crossover_prob", C.c_double),
        ("x0", C.c_void_p),
        ("sigma", C.c_void_p),
        ("inject", C.POINTER(empc_injected)),
        ("u_out", C.c_void_p),
        ("best_out", C.c_void_p),
        ("best_cost", C.c_void_p),
        ("best_index", C.c_void_p),
    ]


class empc_plant(C.Structure):
    _fields_ = [("kind", C.c_int32), ("links", C.c_int32), ("mass", C.c_void_p),
                ("length", C.c_void_p), ("damping", C.c_double), ("gravity", C.c_double)]


_lib = None


def load(path: str | None = None):
    """Load the CUDA library (once).  Raises if it is missing: no fallback.
    ``EMPC_LIB`` overrides the path (experiment builds)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("EMPC_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = C.CDLL(path)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_void_p  # data pointers as void*
    sig = {
        "empc_create": (C.c_int, [C.POINTER(empc_dims), C.POINTER(P)]),
        "empc_destroy": (None, [P]),
        "empc_last_error": (C.c_char_p, [P]),
        "empc_set_schedule": (C.c_int, [P, P, P, D]),
        "empc_set_scorer": (C.c_int, [P, C.c_int32]),
        "empc_set_problems": (C.c_int, [P, I32, I32] + [D] * 9),
        "empc_pop_alloc": (C.c_int, [P, C.POINTER(I32)]),
        "empc_pop_free": (C.c_int, [P, I32]),
        "empc_pop_read": (C.c_int, [P, I32, D, D]),
        "empc_pop_write": (C.c_int, [P, I32, D, D]),
        "empc_run": (C.c_int, [P, C.POINTER(empc_run_args)]),
        "empc_score": (C.c_int, [P, D, I32, D, D]),
        "empc_select": (C.c_int, [P, D, P, P]),
        "empc_expand": (C.c_int, [P, I32, D, D]),
        "empc_time_device": (C.c_int, [P, C.POINTER(empc_run_args), I32, I32, C.POINTER(C.c_float),
                                        C.POINTER(C.c_float), C.POINTER(I32), C.POINTER(I32)]),
        "empc_describe": (C.c_int, [P, C.c_char_p, I32]),
        "empc_num_variants": (C.c_int, [P, C.POINTER(I32)]),
        "empc_set_variant": (C.c_int, [P, I32]),
        "empc_set_occupancy": (C.c_int, [P, I32]),
        "empc_set_tensor_cores": (C.c_int, [P, I32]),
        "empc_set_option": (C.c_int, [P, I32, I32]),
        "empc_philox": (C.c_int, [P, P, I32, P]),
        "empc_shard_setup": (C.c_int, [P, I64, I32, I64, I32, I32]),
        "empc_shard_entry_bytes": (C.c_int, [P, C.POINTER(I64)]),
        "empc_shard_init": (C.c_int, [P, C.POINTER(empc_run_args)]),
        "empc_shard_export": (C.c_int, [P, P]),
        "empc_shard_import": (C.c_int, [P, P, I32, D, D, D, C.POINTER(I64)]),
        "empc_shard_evolve": (C.c_int, [P, C.POINTER(empc_run_args)]),
        "empc_shard_read": (C.c_int, [P, D, D]),
        "empc_get_stream": (C.c_int, [P, C.POINTER(P)]),
        "empc_plant_linearize_discretize": (C.c_int, [C.POINTER(empc_plant), I32, D, D, C.c_double, C.c_double,
                                                      I32, I32, D, D, D]),
        "empc_plant_integrate": (C.c_int, [C.POINTER(empc_plant), I32, D, D, C.c_double, I32, I32, D]),
        "empc_plant_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, handle=None):
    if rc == EMPC_OK:
        return
    msg = _lib.empc_last_error(handle).decode() if _lib is not None else "unknown error"
    if rc == EMPC_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"empc error {rc}: {msg}")


# Data pointers cross the ABI as void*.  The arrays behind them are kept
# alive for the next few hundred conversions, so a temporary such as
# dptr(f64(x)) outlives the call it is passed to.
_keep = collections.deque(maxlen=512)


def dptr(a: np.ndarray) -> int:
    """Address of a C-contiguous array for a void* argument (ctypes converts
    the int); the array is kept alive for the next few hundred conversions."""
    _keep.append(a)
    return a.ctypes.data


iptr = u8ptr = u32ptr = dptr


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Handle:
    """Owning wrapper of an ``empc_handle*``."""

    def __init__(self, n, m, T, p, num_sims, num_parents, instances=1, dense_q=False, precision=EMPC_FP32,
                 device=0):
        self.lib = load()
        self.dims = empc_dims(n, m, T, p, num_sims, num_parents, instances, int(bool(dense_q)), precision, device)
        h = C.c_void_p()
        rc = self.lib.empc_create(C.byref(self.dims), C.byref(h))
        if rc != EMPC_OK:
            msg = self.lib.empc_last_error(None).decode()
            if rc == EMPC_EINVAL:
                raise ValueError(msg)
            raise RuntimeError(f"empc_create failed ({rc}): {msg}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.empc_destroy(self.h)
            self.h = None

    def call(self, name, *args):
        check(getattr(self.lib, name)(self.h, *args), self.h)

    def describe(self) -> str:
        buf = C.create_string_buffer(512)
        self.call("empc_describe", buf, 512)
        return buf.value.decode()

    def num_variants(self) -> int:
        v = C.c_int32()
        self.call("empc_num_variants", C.byref(v))
        return v.value

    def set_variant(self, v: int):
        self.call("empc_set_variant", int(v))

    def set_occupancy(self, ctas_per_sm: int):
        self.call("empc_set_occupancy", int(ctas_per_sm))

    def set_tensor_cores(self, mode: int):
        self.call("empc_set_tensor_cores", int(mode))

    def set_option(self, option: int, value: int):
        self.call("empc_set_option", int(option), int(value))


def philox4x32_10(ctr: np.ndarray, key: np.ndarray) -> np.ndarray:
    """Device Philox4x32-10 (known-answer seam)."""
    lib = load()
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(ctr)
    check(lib.empc_philox(dptr(ctr), dptr(key), ctr.shape[0], dptr(out)))
    return out


def plant_integrate(kind, links, mass, length, damping, gravity, xs, us, dt, substeps, device=0):
    """Batched device RK4 period of the plant (include/empc_b200.h)."""
    import numpy as np

    lib = load()
    mass, length = f64(mass), f64(length)
    pl = empc_plant(kind, links, dptr(mass), dptr(length), float(damping), float(gravity))
    xs, us = f64(xs), f64(us)
    out = np.empty_like(xs)
    rc = lib.empc_plant_integrate(C.byref(pl), xs.shape[0], dptr(xs), dptr(us), float(dt), int(substeps),
                                  int(device), dptr(out))
    if rc != EMPC_OK:
        msg = lib.empc_plant_last_error().decode()
        raise (ValueError if rc == EMPC_EINVAL else RuntimeError)(msg)
    return out


def plant_linearize_discretize(kind, links, mass, length, damping, gravity, xs, us, eps, dt, method, device=0):
    """Batched device linearize + discretize (include/empc_b200.h)."""
    import numpy as np

    lib = load()
    mass, length = f64(mass), f64(length)
    pl = empc_plant(kind, links, dptr(mass), dptr(length), float(damping), float(gravity))
    xs, us = f64(xs), f64(us)
    cnt, n = xs.shape
    m = us.shape[1]
    Ad = np.empty((cnt, n, n))
    Bd = np.empty((cnt, n, m))
    wd = np.empty((cnt, n))
    rc = lib.empc_plant_linearize_discretize(C.byref(pl), cnt, dptr(xs), dptr(us), float(eps), float(dt),
                                             int(method), int(device), dptr(Ad), dptr(Bd), dptr(wd))
    if rc != EMPC_OK:
        msg = lib.empc_plant_last_error().decode()
        raise (ValueError if rc == EMPC_EINVAL else RuntimeError)(msg)
    return Ad, Bd, wd
