"""The Python side of msg_plan_switch / msg_touch (no GPU): windows packed
into the per-context msg_window array, result buffers grown on demand, and the
arrays and structs returned to the caller are copies that a later call does
not overwrite (the buffers are reused across calls)."""
import ctypes as C

import numpy as np

from paper_2512_24637_b200 import _abi


class FakeLib:
    """Stands in for libmsched_b200: reads the packed windows back and fills
    the result pointers with values derived from them."""

    def __init__(self):
        self.calls = []

    def _windows(self, ptr, nw):
        if not nw:
            return []
        arr = (_abi.Window * nw).from_address(ptr)
        return [(w.task, w.c0, w.c1, w.pad) for w in arr]

    def msg_plan_switch(self, h, wptr, nw, reorder, out_p, pages_p, prefix_p, touch_p):
        wins = self._windows(wptr, nw)
        self.calls.append(("plan", wins, reorder))
        ncw = wins[0][2] - wins[0][1]
        out = _abi.SwitchOut.from_address(out_p)
        out.missing, out.nwin, out.populate, out.first_missing = 7 * nw, nw, 3, wins[0][1]
        for i, (t, a, b, _) in enumerate(wins):
            C.c_int64.from_address(pages_p + 8 * i).value = 1000 * t + (b - a)
        for k in range(ncw):
            C.c_int64.from_address(prefix_p + 8 * k).value = k
            C.c_int64.from_address(touch_p + 8 * k).value = 2 * k + 1
        return 0

    def msg_touch(self, h, idx, cmd, evict, wptr, nw, scan_end, write_tags, out_p, pages_p):
        wins = self._windows(wptr, nw) if wptr else []
        self.calls.append(("touch", idx, cmd, evict, wins, scan_end, write_tags))
        out = _abi.TouchOut.from_address(out_p)
        out.missing, out.evicted, out.next_missing = cmd, evict, scan_end
        for i, (t, a, b, _) in enumerate(wins):
            C.c_int64.from_address(pages_p + 8 * i).value = 10 * t + a
        return 0


def _ctx():
    ctx = _abi.Context.__new__(_abi.Context)   # no device: only the marshaling state
    ctx.lib, ctx.h, ctx.h2d_bytes, ctx.d2h_bytes = FakeLib(), None, 0, 0
    ctx._sout, ctx._tout = _abi.SwitchOut(), _abi.TouchOut()
    ctx._sout_p, ctx._tout_p = C.addressof(ctx._sout), C.addressof(ctx._tout)
    ctx._win_cap = ctx._i64_cap = 0
    ctx._grow_scratch(64, 1024)
    return ctx


def test_plan_switch_packs_windows_and_returns_copies():
    ctx = _ctx()
    wins = [(0, 10, 14), (1, 0, 9), (2, 5, 6)]
    out, pages, prefix, touch = ctx.plan_switch(wins, reorder_always=True)
    assert ctx.lib.calls[-1] == ("plan", [(t, a, b, 0) for t, a, b in wins], 1)
    assert out.missing == 21 and out.nwin == 3 and out.first_missing == 10
    assert pages.tolist() == [4, 1009, 2001]
    assert prefix.tolist() == [0, 1, 2, 3] and touch.tolist() == [1, 3, 5, 7]
    # a second call reuses the buffers: the first call's results must not change
    ctx.plan_switch([(3, 0, 2)])
    assert out.missing == 21 and pages.tolist() == [4, 1009, 2001] and prefix.tolist() == [0, 1, 2, 3]


def test_buffers_grow_for_many_windows_and_long_slices():
    ctx = _ctx()
    wins = [(i, 0, 3000 if i == 0 else 2) for i in range(100)]   # > 64 windows, > 1024 slice commands
    out, pages, prefix, touch = ctx.plan_switch(wins)
    assert ctx._win_cap >= 100 and ctx._i64_cap >= 100 + 2 * 3000
    assert ctx.lib.calls[-1][1] == [(t, a, b, 0) for t, a, b in wins]
    assert pages[0] == 3000 and pages[99] == 99002 and len(prefix) == 3000 and touch[-1] == 5999
    # and shrink back to a small call without stale windows leaking in
    ctx.plan_switch([(5, 1, 4)])
    assert ctx.lib.calls[-1][1] == [(5, 1, 4, 0)]


def test_touch_with_and_without_refresh_windows():
    ctx = _ctx()
    out, pages = ctx.touch(2, 17, 0, [], 30, False)
    assert ctx.lib.calls[-1] == ("touch", 2, 17, 0, [], 30, 0) and len(pages) == 0
    assert out.missing == 17 and out.next_missing == 30
    out2, pages2 = ctx.touch(1, 5, 9, [(1, 5, 8), (0, 0, 4)], 8, True)
    assert ctx.lib.calls[-1][4] == [(1, 5, 8, 0), (0, 0, 4, 0)] and ctx.lib.calls[-1][6] == 1
    assert pages2.tolist() == [15, 0] and out2.evicted == 9
    assert out.missing == 17   # the first call's struct is the caller's own copy
    assert isinstance(pages2, np.ndarray) and pages2.dtype == np.int64
