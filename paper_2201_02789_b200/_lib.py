"""ctypes binding of libdynpar.so (include/dynpar.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2201_02789_b200/csrc``).  There is no CPU fallback: if the library is
missing, or no sm_100 device is visible, every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

CSRC = Path(__file__).resolve().parent / "csrc"
LIB_PATH = Path(os.environ.get("DYNPAR_LIB", CSRC / "libdynpar.so"))

AGG_CODES = {None: 0, "none": 0, "warp": 1, "block": 2, "multiblock": 3,
             "grid": 4}
VARIANT_NOCDP, VARIANT_CDP = 0, 1
SERIAL_MODES = {"thread": 0, "warp": 1}
INF_THRESHOLD = 2147483647  # passes/common.py:10

# DP_ERR_* -> SimTrap kinds (sim/machine.py:43-50)
ERROR_KINDS = {-1: "queue-overflow", -2: "launch-config", -3: "cuda-error",
               -4: "invalid-argument", -5: "no-device",
               -6: "iteration-limit", -7: "unpublished-read"}


class DpConfig(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_int32), ("cfactor", ctypes.c_int32),
                ("agg", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("agg_threshold", ctypes.c_int32),
                ("variant", ctypes.c_int32),
                ("parent_block", ctypes.c_int32),
                ("child_block", ctypes.c_int32),
                ("serial_mode", ctypes.c_int32),
                ("pending_launch_limit", ctypes.c_int32),
                ("persistent", ctypes.c_int32),
                ("device_loop", ctypes.c_int32),
                ("frontier", ctypes.c_int32),
                ("agg_coarsen", ctypes.c_int32),
                ("counts_spread", ctypes.c_int32),
                ("weight_bits", ctypes.c_int32),
                ("cf_wave", ctypes.c_int32),
                ("col_bits", ctypes.c_int32)]


class DpStats(ctypes.Structure):
    _fields_ = [("num_launches", ctypes.c_uint64),
                ("host_launches", ctypes.c_uint64),
                ("blocks_scheduled", ctypes.c_uint64),
                ("max_pending_depth", ctypes.c_uint64),
                ("iterations", ctypes.c_uint64),
                ("work_units", ctypes.c_uint64),
                ("bytes_alg", ctypes.c_uint64),
                ("ns_device", ctypes.c_double),
                ("ns_host", ctypes.c_double),
                ("ns_kernel_max", ctypes.c_double),
                ("ns_kernel_sum", ctypes.c_double),
                ("ns_phase", ctypes.c_double * 5),
                ("h2d_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64),
                ("launch_lat_ns_mean", ctypes.c_double),
                ("remote_ops", ctypes.c_uint64),
                ("unpublished_reads", ctypes.c_uint64),
                ("poisoned_reads", ctypes.c_uint64)]


class DeviceTrap(RuntimeError):
    """Runtime fault on the device; mirrors ``dynoptc.sim.SimTrap``
    (sim/machine.py:43-50): ``kind`` uses the same vocabulary."""

    def __init__(self, kind: str, message: str, kernel: str = "",
                 line: int = 0):
        super().__init__(f"{kind}: {message}")
        self.kind = kind
        self.message = message
        self.kernel = kernel
        self.line = line


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_F32 = ctypes.c_float
_CFG = ctypes.POINTER(DpConfig)
_ST = ctypes.POINTER(DpStats)

_SIGNATURES = {
    "dp_abi_version": ([], ctypes.c_int),
    "dp_last_error": ([], ctypes.c_char_p),
    "dp_device_count": ([], ctypes.c_int),
    "dp_init": ([_I32], ctypes.c_int),
    "dp_bfs": ([_P, _P, _I32, _I64, _I32, _CFG, _P, _P, _ST], ctypes.c_int),
    "dp_bfs_dev": ([_P, _P, _I32, _I64, _I32, _CFG, _P, _P, _P, _ST],
                   ctypes.c_int),
    "dp_sssp": ([_P, _P, _P, _I32, _I64, _I32, _CFG, _P, _ST], ctypes.c_int),
    "dp_sssp_dev": ([_P, _P, _P, _I32, _I64, _I32, _CFG, _P, _P, _ST],
                    ctypes.c_int),
    "dp_manylaunch": ([_P, _I32, _CFG, _P, _P, _ST], ctypes.c_int),
    "dp_manylaunch_dev": ([_P, _I32, _CFG, _P, _P, _P, _ST], ctypes.c_int),
    "dp_tc": ([_P, _P, _I32, _I64, _I64, _I64, _CFG, _P, _ST], ctypes.c_int),
    "dp_tc_dev": ([_P, _P, _I32, _I64, _I64, _I64, _CFG, _P, _P, _ST],
                  ctypes.c_int),
    "dp_bt": ([_P, _I32, _I32, _F32, _CFG, _P, _P, _P, _I64, _P, _ST],
              ctypes.c_int),
    "dp_bt_dev": ([_P, _I32, _I32, _F32, _CFG, _P, _P, _P, _I64, _P, _P,
                   _ST], ctypes.c_int),
    "dp_unspread_dev": ([_P, _I32, _I32, _P, _P], _I32),
    "dp_bfs_part_level": ([_P, _P, _I32, _I32, _I32, _I32, _CFG, _P, _P,
                           _P, _P, _I64, _P, _P, _P, _ST], ctypes.c_int),
    "dp_bfs_part_apply": ([_P, _I64, _I32, _I32, _P, _P, _P], ctypes.c_int),
    "dp_bfs_part_level_peer": ([_P, _P, _I32, _I32, _I32, _I32, _CFG, _P, _P,
                                _P, _P, _P, _P, _ST], ctypes.c_int),
    "dp_sssp_part_round": ([_P, _P, _P, _I32, _I32, _I32, _CFG, _P, _P, _P,
                            _P, _P, _P, _P, _ST], ctypes.c_int),
    "dp_sssp_part_apply": ([_P, _I64, _I32, _P, _P, _P], ctypes.c_int),
    "dp_sssp_part_solve_peer": ([_P, _P, _P, _I32, _I32, _I32, _I32, _I32,
                                 _CFG, _P, _P, _P, _P, _U64, _P, _ST],
                                ctypes.c_int),
    "dp_bfs_part_solve_peer": ([_P, _P, _I32, _I32, _I32, _I32, _I32, _CFG,
                                _P, _P, _P, _I64, _P, _P, _U64, _P, _ST],
                               ctypes.c_int),
    "dp_thread_release": ([], None),
    "dp_step_times": ([_P, _I64], _I64),
    "dp_sssp_part_round_peer": ([_P, _P, _P, _I32, _I32, _I32, _CFG, _P, _P,
                                 _P, _P, _P, _ST], ctypes.c_int),
    "dp_rmat_part_keys_dev": ([_I32, _I32, _U64, _I32, _I32, _P, _I64,
                               ctypes.POINTER(ctypes.c_int64), _P],
                              ctypes.c_int),
    "dp_rmat_csr": ([_I32, _I32, _U64, _P, _P, _I32], ctypes.c_int),
    "dp_rmat_csr_part": ([_I32, _I32, _U64, _I32, _I32, _P, _P, _I64,
                          ctypes.POINTER(ctypes.c_int64), _I32],
                         ctypes.c_int),
    "dp_tc_orient": ([_P, _P, _I32, ctypes.POINTER(ctypes.c_void_p),
                      ctypes.POINTER(ctypes.c_void_p),
                      ctypes.POINTER(ctypes.c_int64), _I32], ctypes.c_int),
    "dp_gc": ([_P, _P, _I32, _I64, _CFG, _P, _ST], ctypes.c_int),
    "dp_gc_dev": ([_P, _P, _I32, _I64, _CFG, _P, _P, _ST], ctypes.c_int),
    "dp_symmetrize": ([_P, _P, _I32, ctypes.POINTER(ctypes.c_void_p),
                       ctypes.POINTER(ctypes.c_void_p),
                       ctypes.POINTER(ctypes.c_int64), _I32], ctypes.c_int),
    "dp_mst": ([_P, _P, _P, _P, _I32, _I64, _CFG, _CFG, _P,
                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                _ST], ctypes.c_int),
    "dp_mst_dev": ([_P, _P, _P, _P, _I32, _I64, _CFG, _CFG, _P,
                    ctypes.POINTER(ctypes.c_int64),
                    ctypes.POINTER(ctypes.c_int64), _P, _ST], ctypes.c_int),
    "dp_edge_mirror": ([_P, _P, _I32, _P, _I32], ctypes.c_int),
    "dp_sp": ([_P, _I32, _I32, _P, _P, _I32, _P, _I32, _F32, _CFG, _P, _P,
               _P, ctypes.POINTER(ctypes.c_int32),
               ctypes.POINTER(ctypes.c_float), _ST], ctypes.c_int),
    "dp_sp_dev": ([_P, _I32, _I32, _P, _P, _I32, _I32, _F32, _CFG, _P, _P,
                   _P, ctypes.POINTER(ctypes.c_int32),
                   ctypes.POINTER(ctypes.c_float), _P, _ST], ctypes.c_int),
    "dp_free": ([_P], None),
}

EXPORTED = tuple(_SIGNATURES)

# include/dynpar.h DP_ABI_VERSION: bumped whenever a struct or signature
# changes (2: dp_config.col_bits)
ABI_VERSION = 2

_lock = threading.Lock()
_lib = None
_device_ready = False


def load() -> ctypes.CDLL:
    """Load libdynpar.so (no device needed).  Raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with "
                    f"`python -c 'import __graft_entry__ as g; g.build()'` "
                    f"or `make -C {CSRC}` (there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            # A/B runs of older builds (tools/ab_libs.py) may lack newer
            # entry points; everything else requires every symbol
            partial = os.environ.get("DYNPAR_LIB_PARTIAL") == "1"
            for name, (args, res) in _SIGNATURES.items():
                if partial and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = res
            if not partial and lib.dp_abi_version() != ABI_VERSION:
                raise ImportError(
                    f"{LIB_PATH} has ABI {lib.dp_abi_version()}, this binding "
                    f"expects {ABI_VERSION} (include/dynpar.h DP_ABI_VERSION): "
                    f"rebuild it")
            _lib = lib
        return _lib


def device() -> ctypes.CDLL:
    """The library with the current CUDA device initialised (sm_100a)."""
    global _device_ready
    lib = load()
    if not _device_ready:
        dev = 0
        try:  # follow torch's current device when torch is in use
            import torch
            if torch.cuda.is_available():
                dev = torch.cuda.current_device()
        except Exception:  # noqa: BLE001 - torch is optional here
            pass
        check(lib.dp_init(dev))
        _device_ready = True
    return lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (load().dp_last_error() or b"").decode(errors="replace")
    kind = ERROR_KINDS.get(rc, "cuda-error")
    if kind == "invalid-argument":
        raise ValueError(msg)
    raise DeviceTrap(kind, msg)


def ptr(a) -> int | None:
    """Address of a C-contiguous numpy array or torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays passed to libdynpar must be contiguous")
        return a.ctypes.data
    return a.data_ptr()


def step_times() -> list[float]:
    """Per-step device ms of this thread's last run (dp_step_times)."""
    buf = (ctypes.c_double * 4096)()
    k = load().dp_step_times(buf, 4096)
    return [buf[i] for i in range(min(k, 4096))]


def stats_dict(st: DpStats) -> dict:
    out = {name: getattr(st, name) for name, _ in DpStats._fields_
           if name != "ns_phase"}
    out["ns_phase"] = list(st.ns_phase)
    return out
