"""Error behaviour of the C ABI (include/msched_b200.h: return codes,
msg_last_error), the counterpart of the reference's SimulationError /
ValueError paths: bad arguments are MSG_E_INVAL, pages
outside the dense map MSG_E_DOMAIN, residency violations MSG_E_CAPACITY,
no exception crosses the ABI, and a rejected call leaves the context usable
and unchanged."""

import pytest

from paper_2512_24637_b200 import _abi
from paper_2512_24637_b200._abi import Context, MsgError

pytestmark = pytest.mark.gpu


def code_of(fn, *a):
    with pytest.raises(MsgError) as ei:
        fn(*a)
    assert str(ei.value)          # msg_last_error text travels with the code
    return ei.value.code


@pytest.mark.parametrize("page,cap", [(4095, 16), (0, 16), (4096, 0), (4096, 1 << 31)])
def test_create_rejects_bad_config(page, cap):
    assert code_of(Context, page, cap) == _abi.MSG_E_INVAL


def test_domain_errors_leave_context_unset():
    ctx = Context(4096, 64)
    try:
        assert code_of(ctx.set_domain, [(0, 1 << 31)]) == _abi.MSG_E_DOMAIN
        ctx.set_domain([(100, 200), (150, 300)])      # still settable; overlapping spans merge
        assert code_of(ctx.set_domain, [(0, 10)]) == _abi.MSG_E_INVAL   # only once
        ctx.list_append([(100, 110)])
        assert ctx.list_read().tolist() == list(range(100, 110))
    finally:
        ctx.close()


def test_list_errors_do_not_mutate():
    ctx = Context(4096, 16)
    try:
        ctx.set_domain([(0, 64)])
        ctx.list_append([(0, 10)])
        assert code_of(ctx.list_append, [(60, 70)]) == _abi.MSG_E_DOMAIN      # 64..69 outside the map
        assert code_of(ctx.list_append, [(20, 30)]) == _abi.MSG_E_CAPACITY    # 10 + 10 > 16 frames
        assert ctx.list_read().tolist() == list(range(10))
        ctx.list_madvise([(2, 4)])
        assert ctx.list_read().tolist() == [0, 1, 4, 5, 6, 7, 8, 9, 2, 3]
    finally:
        ctx.close()


def test_unknown_tasks_and_commands_are_inval():
    ctx = Context(4096, 16)
    try:
        ctx.set_domain([(0, 64)])
        assert code_of(ctx.plan_switch, [(3, 0, 1)]) == _abi.MSG_E_INVAL
        assert code_of(ctx.touch, 7, 0, 0, [], 1, False) == _abi.MSG_E_INVAL
        assert code_of(ctx.read_pages, 0, 0, 0) == _abi.MSG_E_INVAL
        ctx.add_task(0, [(0, 8)])
        assert code_of(ctx.add_task, 0, [(0, 8)]) == _abi.MSG_E_INVAL          # registered twice
        assert code_of(ctx.add_task, -1, [(0, 8)]) == _abi.MSG_E_INVAL
        assert code_of(ctx.read_pages, 0, 5, 0) == _abi.MSG_E_INVAL            # no command 5
        assert ctx.list_len() == 0
    finally:
        ctx.close()


def test_bad_ranges_and_negative_counts_are_inval():
    import ctypes as C

    from paper_2512_24637_b200 import engine
    from paper_2512_24637_b200.presets import get_preset
    from paper_2512_24637_b200.scenarios import streaming_scenario

    hw = get_preset("rtx5080").with_capacity(96 << 20)
    tasks, pol = streaming_scenario(hw, 1.5)
    sim = engine.Simulator(tasks, hw, pol, engine.Mode.um())
    try:
        ctx, n0 = sim.ctx, len(tasks[0].commands)
        assert code_of(ctx.um_slice, 0, 0, n0 + 1) == _abi.MSG_E_INVAL
        assert code_of(ctx.um_slice, 0, 2, 1) == _abi.MSG_E_INVAL
        assert code_of(ctx.plan_switch, [(0, 0, 1), (1, 0, 10 ** 6)]) == _abi.MSG_E_INVAL
        lib, h = ctx.lib, ctx.h
        got = C.c_int64()
        assert lib.msg_list_append(h, None, None, -1) == _abi.MSG_E_INVAL
        assert lib.msg_list_read(h, None, -5, C.byref(got)) == _abi.MSG_E_INVAL
        assert lib.msg_release_task(h, None, None, -2, C.byref(got)) == _abi.MSG_E_INVAL
        assert lib.msg_last_error(h).decode() == "negative count"
        m = sim.run()                 # the context is still good after every rejected call
        assert m.completed_tasks == len(tasks)
    finally:
        sim.close()


def test_add_commands_rejects_tables_outside_their_arrays():
    """msg_add_commands copies and reads exactly the windows the command
    table names: negative offsets/counts, raw-struct windows past the blob,
    non-positive range lengths and memcpy extents are MSG_E_INVAL before any
    byte is read, and the task stays usable."""
    import numpy as np

    from paper_2512_24637_b200.model import Arg, ByteRange, Command, CommandKind

    base = 1 << 40
    ctx = Context(4096, 64)
    try:
        ctx.set_domain([(base >> 12, (base >> 12) + 64)])
        ctx.add_task(0, [(base, 64 * 4096)])
        cmds = [Command(CommandKind.KERNEL, 1e-5, "k", (Arg(base, 64), Arg(0, 64, raw=base.to_bytes(8, "little"))),
                        ground_truth_access=(ByteRange(base, 8192),)),
                Command(CommandKind.MEMCPY_H2D, 1e-5, "", (Arg(0), Arg(base), Arg(4096)))]
        good = _abi.encode_commands(cmds, {"k": 0})

        def mutated(fn):
            c, a, b, bl, g = (x.copy() if isinstance(x, np.ndarray) else x for x in good)
            fn(c, a, b, g)
            return c, a, b, bl, g

        bad = [
            lambda c, a, b, g: c["arg_off"].__setitem__(0, -1),
            lambda c, a, b, g: c["ngt"].__setitem__(0, -1),
            lambda c, a, b, g: a["raw_off"].__setitem__(1, 4),           # 8-byte window at 4 of an 8-byte blob
            lambda c, a, b, g: a["raw_off"].__setitem__(1, -8),
            lambda c, a, b, g: g["len"].__setitem__(0, 0),
            lambda c, a, b, g: g["len"].__setitem__(0, -4096),
            lambda c, a, b, g: c["dev_len"].__setitem__(1, 0),
            lambda c, a, b, g: c["kind"].__setitem__(0, 5),
        ]
        for fn in bad:
            assert code_of(ctx.add_commands, 0, mutated(fn)) == _abi.MSG_E_INVAL
        ctx.add_commands(0, good)                # the untouched tables still go in
        assert ctx.read_pages(0, 0, 1) == [(base >> 12, (base >> 12) + 2)]
    finally:
        ctx.close()
