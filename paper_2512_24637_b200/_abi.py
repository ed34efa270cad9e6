"""ctypes binding of libmsched_b200.so (include/msched_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, `load()` raises.  Struct layouts mirror the C header and
are checked by tests/test_abi.py.
"""

from __future__ import annotations

import ctypes as C
import os
import struct
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmsched_b200.so")

MSG_OK, MSG_E_INVAL, MSG_E_DOMAIN, MSG_E_CAPACITY, MSG_E_OOM, MSG_E_CUDA = 0, -1, -2, -3, -4, -5
PRED_TEMPLATE, PRED_ALLOCATION, PRED_TRUTH = 0, 1, 2
CMD_KERNEL, CMD_H2D, CMD_D2H = 0, 1, 2
F_MIGRATE, F_VERIFY_TAGS, F_LOOSE_DOMAIN, F_EXECUTE = 1, 2, 4, 8

EXPORTS = [
    "msg_create", "msg_destroy", "msg_last_error", "msg_stream", "msg_set_domain", "msg_add_task",
    "msg_set_rules", "msg_add_commands", "msg_read_pages", "msg_read_pages_range", "msg_plan_switch", "msg_touch",
    "msg_um_slice", "msg_release_task", "msg_list_append", "msg_list_madvise", "msg_list_evict_head",
    "msg_list_len", "msg_list_read", "msg_sync", "msg_get_stats", "msg_verify_residency",
    "msg_flush_l2", "msg_list_reorder", "msg_debug", "msg_debug_read", "msg_window_runs", "msg_list_plan", "msg_reset",
    "msg_run_command", "msg_analyze",
]


class MsgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Cfg(C.Structure):
    _fields_ = [("device", C.c_int32), ("predictor", C.c_int32), ("page_size", C.c_int64),
                ("capacity_pages", C.c_int64), ("host_pool_pages", C.c_int64), ("flags", C.c_uint32),
                ("reserved", C.c_uint32)]


class Window(C.Structure):
    _fields_ = [("task", C.c_int32), ("c0", C.c_int32), ("c1", C.c_int32), ("pad", C.c_int32)]


class SwitchOut(C.Structure):
    _fields_ = [("missing", C.c_int64), ("early_exit", C.c_int32), ("nwin", C.c_int32),
                ("populate", C.c_int64), ("evict", C.c_int64), ("truncated", C.c_int64),
                ("free_before", C.c_int64), ("resident_after", C.c_int64), ("first_missing", C.c_int32),
                ("pad", C.c_int32), ("first_missing_pages", C.c_int64)]


class TouchOut(C.Structure):
    _fields_ = [("missing", C.c_int64), ("evicted", C.c_int64), ("resident_after", C.c_int64),
                ("refreshed", C.c_int32), ("next_missing", C.c_int32), ("next_missing_pages", C.c_int64)]


class Stats(C.Structure):
    _fields_ = [("kernels", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("h2d_segments", C.c_int64), ("d2h_segments", C.c_int64), ("ce_batches", C.c_int64),
                ("sm_batches", C.c_int64), ("h2d_busy_ms", C.c_double), ("d2h_busy_ms", C.c_double),
                ("plan_ms", C.c_double), ("ms_passes", C.c_int64), ("ms_ms", C.c_double),
                ("ms_bytes", C.c_int64), ("run_cmds", C.c_int64), ("run_pages", C.c_int64),
                ("run_bad_tags", C.c_int64), ("run_missing", C.c_int64), ("run_ms", C.c_double),
                ("ms_dev_launches", C.c_int64), ("ms_dev_ms", C.c_double),
                ("ms_ev_passes", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


ARG_DT = np.dtype([("lo", "<u8"), ("hi", "<i8"), ("width", "<i4"), ("raw_len", "<i4"), ("raw_off", "<i8")])
CMD_DT = np.dtype([("kind", "<i4"), ("kernel", "<i4"), ("arg_off", "<i4"), ("nargs", "<i4"), ("gt_off", "<i4"),
                   ("ngt", "<i4"), ("dims", "<i8", (6,)), ("dev_addr", "<i8"), ("dev_len", "<i8")])
RANGE_DT = np.dtype([("start", "<i8"), ("len", "<i8")])
EXPR_DT = np.dtype([("num", "<i8"), ("den", "<i8"), ("nslots", "<i4"), ("pad", "<i4"), ("slot", "<i8", (3,))])
RULE_DT = np.dtype([("kind", "<i4"), ("ptr_arg", "<i4"), ("offset", "<i8"), ("e", EXPR_DT, (3,))])
ARULE_DT = np.dtype([("ptr_arg", "<i4"), ("kind", "<i4"), ("offset", "<i8"), ("nslots", "<i4", (3,)), ("pad", "<i4"),
                     ("slot", "<i8", (3, 3)), ("v0", "<i8", (3,))])

_lib = None
_WIN_PACK = struct.Struct("<4i").pack_into   # one msg_window


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def load():
    """Load the C-ABI library; raise loudly when it (or a GPU) is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "msg_create": ([C.POINTER(Cfg), C.POINTER(vp)], C.c_int),
        "msg_destroy": ([vp], None),
        "msg_last_error": ([vp], C.c_char_p),
        "msg_stream": ([vp], vp),
        "msg_set_domain": ([vp, vp, vp, i32], C.c_int),
        "msg_add_task": ([vp, i32, vp, i32], C.c_int),
        "msg_set_rules": ([vp, i32, vp, vp, i32], C.c_int),
        "msg_add_commands": ([vp, i32, i32, vp, vp, vp, i64, vp, vp], C.c_int),
        "msg_read_pages": ([vp, i32, i32, i32, vp, i64, C.POINTER(i64)], C.c_int),
        "msg_read_pages_range": ([vp, i32, i32, i32, i32, vp, i64, vp, C.POINTER(i64)], C.c_int),
        "msg_plan_switch": ([vp, vp, i32, i32, vp, vp, vp, vp], C.c_int),
        "msg_touch": ([vp, i32, i32, i64, vp, i32, i32, i32, vp, vp], C.c_int),
        "msg_um_slice": ([vp, i32, i32, i32, vp, vp], C.c_int),
        "msg_release_task": ([vp, vp, vp, i32, C.POINTER(i64)], C.c_int),
        "msg_list_append": ([vp, vp, vp, i32], C.c_int),
        "msg_list_madvise": ([vp, vp, vp, i32], C.c_int),
        "msg_list_evict_head": ([vp, i64, vp, C.POINTER(i64)], C.c_int),
        "msg_list_len": ([vp, C.POINTER(i64)], C.c_int),
        "msg_list_read": ([vp, vp, i64, C.POINTER(i64)], C.c_int),
        "msg_list_reorder": ([vp, vp, vp, vp, i32, i32, vp], C.c_int),
        "msg_window_runs": ([vp, vp, vp, vp, i32, i32, vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "msg_list_plan": ([vp, vp, vp, i32, i64, vp, C.POINTER(i64), vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "msg_debug": ([vp, i32], C.c_int),
        "msg_reset": ([vp, i32], C.c_int),
        "msg_debug_read": ([vp, i32, vp, i64, C.POINTER(i64)], C.c_int),
        "msg_sync": ([vp], C.c_int),
        "msg_get_stats": ([vp, C.POINTER(Stats)], C.c_int),
        "msg_verify_residency": ([vp, C.POINTER(i64)], C.c_int),
        "msg_flush_l2": ([vp], C.c_int),
        "msg_run_command": ([vp, i32, i32, i64, C.c_double], C.c_int),
        "msg_analyze": ([vp, i32, vp, vp, i64, vp, vp, i32, vp, vp, vp, vp, i32, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def cuda_device_count() -> int:
    try:
        rt = C.CDLL("libcudart.so")
    except OSError:
        import glob

        cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        if not cands:
            return 0
        rt = C.CDLL(cands[0])
    n = C.c_int(0)
    if rt.cudaGetDeviceCount(C.byref(n)) != 0:
        return 0
    return n.value


# ---------------------------------------------------------------------------
# slot codes and rule lowering (analyzer.py:78-96 slot names)

_DIMS = {"gx": 0, "gy": 1, "gz": 2, "bx": 3, "by": 4, "bz": 5}


def slot_code(name: str) -> int:
    if name in _DIMS:
        return 2 | (_DIMS[name] << 2)
    if not name.startswith("a"):
        raise ValueError(f"bad slot {name!r}")
    head, _, tail = name[1:].partition("+")
    idx = int(head)
    if not tail:
        return idx << 2
    off, w = tail.split("w")
    return 1 | (idx << 2) | (int(off) << 18) | ((1 if int(w) == 64 else 0) << 50)


_NEVER = 2 | (7 << 2)   # launch dim 7 does not exist: evaluates to None
_DIM_NAMES = ("gx", "gy", "gz", "bx", "by", "bz")


def slot_name(code: int) -> str:
    """Inverse of slot_code."""
    kind, idx = code & 3, (code >> 2) & 0xFFFF
    if kind == 2:
        return _DIM_NAMES[idx]
    if kind == 0:
        return f"a{idx}"
    return f"a{idx}+{(code >> 18) & 0xFFFFFFFF}w{64 if (code >> 50) & 1 else 32}"


def analyze(cmds_encoded, latency, nkernels: int):
    """msg_analyze over encoded commands (cmds[i].kernel = kernel-name index).
    Returns (status, latency_mean, unpredictable, rules ARULE_DT, rule_off)."""
    lib = load()
    carr, aarr, barr, blen, garr = cmds_encoded
    lat = np.ascontiguousarray(latency, dtype=np.float64)
    status = np.zeros(max(nkernels, 1), np.int32)
    lat_out = np.zeros(max(nkernels, 1), np.float64)
    unp = np.zeros(max(nkernels, 1), np.float64)
    off = np.zeros(nkernels + 1, np.int32)
    cap = max(4 * nkernels, 16)
    while True:
        rules = np.zeros(cap, ARULE_DT)
        rc = lib.msg_analyze(_p(carr), len(carr), _p(aarr), _p(barr), blen, _p(garr), _p(lat), nkernels, _p(status),
                             _p(lat_out), _p(unp), _p(rules), cap, _p(off))
        if rc == MSG_OK:
            return status[:nkernels], lat_out[:nkernels], unp[:nkernels], rules, off
        if rc == MSG_E_INVAL and off[nkernels] > cap:
            cap = int(off[nkernels])
            continue
        raise MsgError(rc, f"msg_analyze failed ({rc})")


def _fits64(v: int) -> bool:
    return -(1 << 63) <= v < (1 << 63)


def lower_expr(e, out):
    coeff = Fraction(e.coeff)
    if not (_fits64(coeff.numerator) and _fits64(coeff.denominator)):
        raise MsgError(MSG_E_DOMAIN, f"coefficient {coeff} exceeds 64 bits")
    out["num"], out["den"] = coeff.numerator, coeff.denominator
    out["nslots"] = len(e.slots)
    if len(e.slots) > 3:
        raise MsgError(MSG_E_DOMAIN, "more than 3 product terms")
    for k, s in enumerate(e.slots):
        out["slot"][k] = slot_code(s)


def lower_rules(descriptors: dict):
    """descriptors (kernel name -> KernelDescriptor) -> (names, rule array,
    per-kernel offsets, per-kernel 'incomplete' flag)."""
    names = list(descriptors)
    rows = []
    offs = [0]
    lossy = []
    for nm in names:
        d = descriptors[nm]
        for r in d.rules:
            row = np.zeros((), RULE_DT)
            row["ptr_arg"] = r.ptr_arg_index
            row["offset"] = r.offset_bytes
            if r.kind in ("fixed", "linear"):
                row["kind"] = 0
                lower_expr(r.size, row["e"][0])
            elif r.kind == "strided":
                row["kind"] = 1
                for k, e in enumerate((r.stride, r.chunk, r.count)):
                    lower_expr(e, row["e"][k])
            else:  # unpredictable: never evaluates (analyzer.py:158-159)
                row["kind"] = 0
                row["e"][0]["den"] = 1
                row["e"][0]["nslots"] = 1
                row["e"][0]["slot"][0] = _NEVER
            rows.append(row)
        offs.append(len(rows))
        lossy.append(d.unpredictable_fraction > 0.0)
    arr = np.array(rows, dtype=RULE_DT) if rows else np.zeros(1, RULE_DT)
    return names, arr, np.asarray(offs, dtype=np.int32), lossy


def _split128(v: int):
    hi = v >> 64
    if not _fits64(hi):
        raise MsgError(MSG_E_DOMAIN, f"argument value {v} exceeds 128 bits")
    return v & 0xFFFFFFFFFFFFFFFF, hi


_KIND_CODE = {"KERNEL": CMD_KERNEL, "H2D": CMD_H2D, "D2H": CMD_D2H}


def encode_commands(cmds, kernel_ids: dict):
    """Columnarise Command objects into the C structs (one pass, host; rows
    built as tuples and converted once)."""
    rows, args, gts, blob = [], [], [], bytearray()
    kid = kernel_ids.get
    for c in cmds:
        kind = c.kind.value if hasattr(c.kind, "value") else c.kind
        code = _KIND_CODE[kind]
        a0, g0 = len(args), len(gts)
        for a in c.launch_args:
            v = a.value
            if -(1 << 63) <= v < (1 << 63):
                lo, hi = v & 0xFFFFFFFFFFFFFFFF, -1 if v < 0 else 0
            else:
                lo, hi = _split128(v)
            if a.raw is not None:
                args.append((lo, hi, 0, len(a.raw), len(blob)))
                blob += a.raw
            else:
                args.append((lo, hi, a.width, -1, 0))
        for r in c.ground_truth_access:
            gts.append((r.start_addr, r.length_bytes))
        if code != CMD_KERNEL:
            rng = c.device_range()   # raises ValueError for non-positive sizes (core.py:52-54)
            da, dl = rng.start_addr, rng.length_bytes
        else:
            da = dl = 0
        rows.append((code, kid(c.kernel_name, -1), a0, len(c.launch_args), g0, len(c.ground_truth_access),
                     tuple(c.grid_dims) + tuple(c.block_dims), da, dl))
    carr = np.array(rows, dtype=CMD_DT) if rows else np.zeros(0, CMD_DT)
    aarr = np.array(args, dtype=ARG_DT) if args else np.zeros(1, ARG_DT)
    garr = np.array(gts, dtype=RANGE_DT) if gts else np.zeros(1, RANGE_DT)
    barr = np.frombuffer(bytes(blob) or b"\0", dtype=np.uint8)
    return carr, aarr, barr, len(blob), garr


class Context:
    """One msg_ctx: one simulated oversubscribed GPU on one CUDA device."""

    def __init__(self, page_size, capacity_pages, predictor=PRED_TRUTH, device=0, flags=0, host_pool_pages=0):
        self.lib = load()
        if cuda_device_count() < 1:
            raise RuntimeError("no CUDA device visible: the proactive memory-scheduling path runs on a B200 "
                               "(there is no CPU fallback)")
        cfg = Cfg(device, predictor, page_size, capacity_pages, host_pool_pages, flags, 0)
        h = C.c_void_p()
        rc = self.lib.msg_create(C.byref(cfg), C.byref(h))
        if rc != 0:
            raise MsgError(rc, f"msg_create failed ({rc})")
        self.h = h
        self.page_size = page_size
        self.capacity = capacity_pages
        self.h2d_bytes = 0   # host->device bytes handed to the ABI (inputs)
        self.d2h_bytes = 0   # device->host result bytes read back
        # plan_switch / touch marshal through buffers allocated once per
        # context with their addresses cached (a per-call ctypes array,
        # numpy allocations and .ctypes conversions cost ~20 us per call)
        self._sout, self._tout = SwitchOut(), TouchOut()
        self._sout_p, self._tout_p = C.addressof(self._sout), C.addressof(self._tout)
        self._win_cap = 0
        self._i64_cap = 0
        self._grow_scratch(64, 1024)

    def _grow_scratch(self, nwin, n64):
        if nwin > self._win_cap:
            self._win_cap = max(nwin, 2 * self._win_cap)
            self._warr = (Window * self._win_cap)()
            self._warr_p = C.addressof(self._warr)
            self._wview = memoryview(self._warr).cast("B")
        if n64 > self._i64_cap:
            self._i64_cap = max(n64, 2 * self._i64_cap)
            self._i64 = np.zeros(self._i64_cap, dtype=np.int64)
            self._i64_p = self._i64.ctypes.data

    def _pack_windows(self, windows):
        nw = len(windows)
        if nw > self._win_cap:
            self._grow_scratch(nw, 0)
        mv = self._wview
        for i, (t, a, b) in enumerate(windows):
            _WIN_PACK(mv, 16 * i, t, a, b, 0)
        return nw

    def close(self):
        if getattr(self, "h", None):
            self.lib.msg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc != 0:
            msg = self.lib.msg_last_error(self.h).decode()
            raise MsgError(rc, msg)

    def stream(self) -> int:
        return self.lib.msg_stream(self.h) or 0

    def set_domain(self, spans):
        first = np.asarray([a for a, _ in spans], dtype=np.int64)
        npages = np.asarray([b - a for a, b in spans], dtype=np.int64)
        self.check(self.lib.msg_set_domain(self.h, _p(first), _p(npages), len(spans)))

    def add_task(self, idx, allocs):
        arr = np.array([(a, n) for a, n in allocs], dtype=RANGE_DT) if allocs else np.zeros(1, RANGE_DT)
        self.check(self.lib.msg_add_task(self.h, idx, _p(arr), len(allocs)))

    def set_rules(self, idx, rules, offs):
        self.check(self.lib.msg_set_rules(self.h, idx, _p(rules), _p(offs), len(offs) - 1))

    def add_commands(self, idx, encoded):
        carr, aarr, barr, blen, garr = encoded
        n = len(carr)
        self.h2d_bytes += carr.nbytes + aarr.nbytes + blen + garr.nbytes
        self.d2h_bytes += n
        comp = np.zeros(max(n, 1), dtype=np.uint8)
        if n:
            self.check(self.lib.msg_add_commands(self.h, idx, n, _p(carr), _p(aarr), _p(barr), blen, _p(garr),
                                                 _p(comp)))
        return comp[:n]

    def read_pages(self, idx, cmd, which):
        n = C.c_int64()
        self.check(self.lib.msg_read_pages(self.h, idx, cmd, which, None, 0, C.byref(n)))
        buf = np.zeros(max(2 * n.value, 2), dtype=np.int64)
        self.check(self.lib.msg_read_pages(self.h, idx, cmd, which, _p(buf), n.value, C.byref(n)))
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n.value)]

    def read_pages_range(self, idx, c0, c1, which):
        """Runs of commands [c0, c1) in one copy: (runs int64[n, 2], off int64[c1 - c0 + 1])."""
        n = C.c_int64()
        off = np.zeros(c1 - c0 + 1, dtype=np.int64)
        self.check(self.lib.msg_read_pages_range(self.h, idx, c0, c1, which, None, 0, _p(off), C.byref(n)))
        buf = np.zeros(max(2 * n.value, 2), dtype=np.int64)
        if n.value:
            self.check(self.lib.msg_read_pages_range(self.h, idx, c0, c1, which, _p(buf), n.value, None,
                                                     C.byref(n)))
        return buf[:2 * n.value].reshape(-1, 2), off

    def plan_switch(self, windows, reorder_always=False):
        """msg_plan_switch; returns (SwitchOut, per-window pages, per-command
        gating counts, per-command touch counts), all owned by the caller."""
        if not windows:
            raise MsgError(MSG_E_INVAL, "need at least one window")
        nw = self._pack_windows(windows)
        ncw = windows[0][2] - windows[0][1]
        n64 = nw + 2 * max(ncw, 1)
        if n64 > self._i64_cap:
            self._grow_scratch(0, n64)
        p = self._i64_p
        self.h2d_bytes += 16 * nw
        self.d2h_bytes += C.sizeof(SwitchOut) + 8 * nw + 2 * 8 * ncw
        rc = self.lib.msg_plan_switch(self.h, self._warr_p, nw, int(reorder_always), self._sout_p, p,
                                      p + 8 * nw, p + 8 * (nw + max(ncw, 1)))
        if rc:
            self.check(rc)
        buf = self._i64[:n64].copy()
        o = nw + max(ncw, 1)
        return SwitchOut.from_buffer_copy(self._sout), buf[:nw], buf[nw:nw + ncw], buf[o:o + ncw]

    def touch(self, idx, cmd, evict, windows, scan_end, write_tags):
        """msg_touch; returns (TouchOut, per-window pages of the refresh),
        owned by the caller."""
        nw = self._pack_windows(windows)
        if nw > self._i64_cap:
            self._grow_scratch(0, nw)
        self.h2d_bytes += 16 * nw
        self.d2h_bytes += C.sizeof(TouchOut) + 8 * nw
        rc = self.lib.msg_touch(self.h, idx, cmd, evict, self._warr_p if nw else None, nw, scan_end,
                                int(write_tags), self._tout_p, self._i64_p)
        if rc:
            self.check(rc)
        return TouchOut.from_buffer_copy(self._tout), self._i64[:nw].copy()

    def run_command(self, idx, cmd, need_pages, latency_s=0.0):
        """Execute a command on the device once `need_pages` of the current
        switch's populate have landed (early-start gating); it reads its
        pages and occupies the GPU for its profiled latency."""
        self.check(self.lib.msg_run_command(self.h, idx, cmd, int(need_pages), float(latency_s)))

    def um_slice(self, idx, c0, c1):
        n = c1 - c0
        miss = np.zeros(max(n, 1), dtype=np.int64)
        ev = np.zeros(max(n, 1), dtype=np.int64)
        self.check(self.lib.msg_um_slice(self.h, idx, c0, c1, _p(miss), _p(ev)))
        return miss[:n], ev[:n]

    def release(self, spans):
        f = np.asarray([a for a, _ in spans] or [0], dtype=np.int64)
        e = np.asarray([b for _, b in spans] or [0], dtype=np.int64)
        removed = C.c_int64()
        self.check(self.lib.msg_release_task(self.h, _p(f), _p(e), len(spans), C.byref(removed)))
        return removed.value

    def list_append(self, runs):
        f = np.asarray([a for a, _ in runs] or [0], dtype=np.int64)
        e = np.asarray([b for _, b in runs] or [0], dtype=np.int64)
        self.check(self.lib.msg_list_append(self.h, _p(f), _p(e), len(runs)))

    def list_madvise(self, runs):
        f = np.asarray([a for a, _ in runs] or [0], dtype=np.int64)
        e = np.asarray([b for _, b in runs] or [0], dtype=np.int64)
        self.check(self.lib.msg_list_madvise(self.h, _p(f), _p(e), len(runs)))

    def list_reorder(self, windows_runs):
        """windows_runs: per window, its first-access-ordered runs."""
        f, e, w = [], [], []
        for k, runs in enumerate(windows_runs):
            for a, b in runs:
                f.append(a); e.append(b); w.append(k)
        nw = len(windows_runs)
        pages = np.zeros(max(nw, 1), dtype=np.int64)
        fa = np.asarray(f or [0], dtype=np.int64)
        ea = np.asarray(e or [0], dtype=np.int64)
        wa = np.asarray(w or [0], dtype=np.int32)
        self.check(self.lib.msg_list_reorder(self.h, _p(fa), _p(ea), _p(wa), len(f), nw, _p(pages)))
        return pages[:nw]

    def list_evict_head(self, n):
        out = np.zeros(max(n, 1), dtype=np.int64)
        got = C.c_int64()
        self.check(self.lib.msg_list_evict_head(self.h, n, _p(out), C.byref(got)))
        return out[:got.value]

    def list_len(self):
        n = C.c_int64()
        self.check(self.lib.msg_list_len(self.h, C.byref(n)))
        return n.value

    def list_read(self):
        n = self.list_len()
        out = np.zeros(max(n, 1), dtype=np.int64)
        got = C.c_int64()
        self.check(self.lib.msg_list_read(self.h, _p(out), n, C.byref(got)))
        return out[:got.value]

    def window_runs(self, per_cmd_runs):
        """per_cmd_runs: list (per command) of normalised runs -> ([(a, b, cmd)], pages)."""
        f, e, k = [], [], []
        for ci, runs in enumerate(per_cmd_runs):
            for a, b in runs:
                f.append(a); e.append(b); k.append(ci)
        n = len(f)
        fa = np.asarray(f or [0], dtype=np.int64)
        ea = np.asarray(e or [0], dtype=np.int64)
        ka = np.asarray(k or [0], dtype=np.int32)
        out = np.zeros(3 * max(2 * n, 1), dtype=np.int64)
        nr, pages = C.c_int64(), C.c_int64()
        self.check(self.lib.msg_window_runs(self.h, _p(fa), _p(ea), _p(ka), n, len(per_cmd_runs), _p(out),
                                            C.byref(nr), C.byref(pages)))
        return [(int(out[3 * i]), int(out[3 * i + 1]), int(out[3 * i + 2])) for i in range(nr.value)], pages.value

    def list_plan(self, runs, capacity):
        f = np.asarray([a for a, _ in runs] or [0], dtype=np.int64)
        e = np.asarray([b for _, b in runs] or [0], dtype=np.int64)
        want = sum(b - a for a, b in runs)
        pop = np.zeros(max(min(want, capacity), 1), dtype=np.int64)
        ev = np.zeros(max(self.list_len(), 1), dtype=np.int64)
        npop, nev, trunc = C.c_int64(), C.c_int64(), C.c_int64()
        self.check(self.lib.msg_list_plan(self.h, _p(f), _p(e), len(runs), capacity, _p(pop), C.byref(npop),
                                          _p(ev), C.byref(nev), C.byref(trunc)))
        return pop[:npop.value], ev[:nev.value], trunc.value

    def debug(self, on=True):
        self.check(self.lib.msg_debug(self.h, int(on)))

    def debug_read(self, which):
        n = C.c_int64()
        self.check(self.lib.msg_debug_read(self.h, which, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.int64)
        self.check(self.lib.msg_debug_read(self.h, which, _p(out), n.value, C.byref(n)))
        return out[:n.value]

    def reset(self, keep_tasks=True):
        self.check(self.lib.msg_reset(self.h, int(keep_tasks)))

    def sync(self):
        self.check(self.lib.msg_sync(self.h))

    def stats(self):
        s = Stats()
        self.check(self.lib.msg_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def verify(self):
        bad = C.c_int64()
        self.check(self.lib.msg_verify_residency(self.h, C.byref(bad)))
        return bad.value

    def flush_l2(self):
        self.check(self.lib.msg_flush_l2(self.h))
