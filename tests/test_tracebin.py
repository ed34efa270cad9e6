"""MSIM-TRACE-BIN v1 on the CPU: lossless
round trips against the reference's own trace objects and text format, and
the columns are byte-identical to what the C ABI receives from
`encode_commands` (so the device sees the same tables either way)."""

import dataclasses

import numpy as np
import pytest

from paper_2512_24637_b200 import _abi, engine, tracebin
from paper_2512_24637_b200.model import Task
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import llm_scenario, streaming_scenario
from paper_2512_24637_b200.workload import gen_template_corpus, load_trace, save_trace

HW = get_preset("rtx5080").with_capacity(96 << 20)


def _tasks():
    out = list(llm_scenario(HW, 2.0, n_tasks=2, layers=4, decode_steps=3)[0])
    out += list(streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)[0])[:2]
    corpus = gen_template_corpus(12, seed=3).task            # raw struct args, planted rules
    out.append(Task(id="corpus", allocations=corpus.allocations, commands=corpus.commands, priority=3,
                    arrival_s=0.25))
    return out


def test_round_trip_is_lossless(tmp_path):
    tasks = _tasks()
    p = tmp_path / "t.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    back = tracebin.load_trace_bin(str(p))
    assert [t.id for t in back] == [t.id for t in tasks]
    for a, b in zip(tasks, back):
        assert b.allocations == a.allocations
        assert (b.priority, b.arrival_s) == (a.priority, a.arrival_s)
        assert len(b.commands) == len(a.commands)
        assert list(b.commands) == list(a.commands)
    # a binary trace of columnar tasks re-saves to the same bytes
    q = tmp_path / "u.msimb"
    tracebin.save_trace_bin(back, str(q))
    assert q.read_bytes() == p.read_bytes()


def test_text_v1_converts(tmp_path):
    tasks = _tasks()[:3]
    paths = []
    for i, t in enumerate(tasks):
        pth = tmp_path / f"t{i}.trace"
        save_trace(t, str(pth))
        paths.append(str(pth))
    out = tmp_path / "all.msimb"
    tracebin.trace_v1_to_bin(paths, str(out))
    back = tracebin.load_trace_bin(str(out))
    for pth, b in zip(paths, back):
        assert list(b.commands) == list(load_trace(pth).commands)


def test_columns_equal_the_abi_encoding(tmp_path):
    tasks = _tasks()
    p = tmp_path / "t.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    for a, b in zip(tasks, tracebin.load_trace_bin(str(p))):
        names = sorted({c.kernel_name for c in a.commands if c.kernel_name})
        kid = {n: i * 7 % 5 for i, n in enumerate(names)}          # any rule-table numbering
        for lo, hi in ((0, len(a.commands)), (1, max(1, len(a.commands) // 2))):
            want = _abi.encode_commands(a.commands[lo:hi], kid)
            got = tracebin.encode_columns(b.commands, kid, lo, hi)
            assert np.array_equal(got[0], want[0])
            n_args, n_gt = int(want[0]["nargs"].sum()), int(want[0]["ngt"].sum())
            assert np.array_equal(got[1][:n_args], want[1][:n_args])
            assert np.array_equal(got[4][:n_gt], want[4][:n_gt])
            for row in want[0]:   # raw-struct bytes behind every argument
                for arg_w, arg_g in zip(want[1][row["arg_off"]:row["arg_off"] + row["nargs"]],
                                        got[1][row["arg_off"]:row["arg_off"] + row["nargs"]]):
                    if arg_w["raw_len"] >= 0:
                        assert bytes(got[2][arg_g["raw_off"]:arg_g["raw_off"] + arg_g["raw_len"]]) == \
                            bytes(want[2][arg_w["raw_off"]:arg_w["raw_off"] + arg_w["raw_len"]])


def test_domain_spans_match(tmp_path):
    tasks = _tasks()
    p = tmp_path / "t.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    back = tracebin.load_trace_bin(str(p))
    assert sorted(engine.domain_spans(back, 4096)) == sorted(engine.domain_spans(tasks, 4096))


def test_corrupt_files_are_rejected(tmp_path):
    p = tmp_path / "bad.msimb"
    p.write_bytes(b"NOTATRACE" + b"\0" * 64)
    with pytest.raises(tracebin.TraceBinError):
        tracebin.load_trace_bin(str(p))
    good = tmp_path / "good.msimb"
    tracebin.save_trace_bin(_tasks()[:1], str(good))
    data = bytearray(good.read_bytes())
    data[12:14] = b"{{"
    p.write_bytes(bytes(data))
    with pytest.raises(tracebin.TraceBinError):
        tracebin.load_trace_bin(str(p))


def test_lazy_commands_support_the_reference_api(tmp_path):
    tasks = _tasks()[:1]
    p = tmp_path / "t.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    b = tracebin.load_trace_bin(str(p))[0]
    assert b.commands[-1] == tasks[0].commands[-1]
    assert b.commands[1:3] == tasks[0].commands[1:3]
    assert dataclasses.replace(b, cursor=2).remaining() == len(tasks[0].commands) - 2


def _corrupt(tmp_path, mutate):
    """Write a valid trace, load its columns, mutate them, re-save through
    the columnar path and load again: the loader must reject it."""
    from paper_2512_24637_b200.model import Allocation, Arg, ByteRange, Command, CommandKind

    base = 1 << 40
    raw = Task(id="raw", allocations=[Allocation("raw.a", base, 1 << 20, "raw")],
               commands=[Command(CommandKind.KERNEL, 1e-5, f"k{i % 2}",
                                 (Arg(base, 64), Arg(0, 64, raw=(base + 4096 * i).to_bytes(8, "little") * 2)),
                                 ground_truth_access=(ByteRange(base + 4096 * i, 4096),)) for i in range(6)])
    p = tmp_path / "ok.msimb"
    tracebin.save_trace_bin(_tasks() + [raw], str(p))
    back = tracebin.load_trace_bin(str(p))
    # a task with raw struct args when there is one (the struct-arg tasks)
    t = max(back, key=lambda x: (int((x.commands.args["raw_len"] >= 0).sum()), len(x.commands)))
    c = t.commands
    cols = tracebin.CommandColumns(c.cmds.copy(), c.args.copy(), c.blob.copy(), c.gts.copy(), c.lat.copy(),
                                   list(c.names))
    mutate(cols)
    q = tmp_path / "bad.msimb"
    bad = tracebin.ColumnarTask(id=t.id, allocations=t.allocations, commands=cols, priority=t.priority,
                                arrival_s=t.arrival_s)
    tracebin.save_trace_bin([bad], str(q))
    with pytest.raises(tracebin.TraceBinError):
        tracebin.load_trace_bin(str(q))


def _first_raw(cols):
    return int(np.flatnonzero(cols.args["raw_len"] >= 0)[0])


@pytest.mark.parametrize("name,mutate", [
    ("arg_off past the table", lambda c: c.cmds["arg_off"].__setitem__(-1, len(c.args) + 5)),
    ("negative nargs", lambda c: c.cmds["nargs"].__setitem__(0, -1)),
    ("gt runs overlap", lambda c: c.cmds["gt_off"].__setitem__(1, 0)),
    ("raw window past the blob",
     lambda c: c.args["raw_off"].__setitem__(_first_raw(c), len(c.blob))),
    ("negative raw offset", lambda c: c.args["raw_off"].__setitem__(_first_raw(c), -8)),
    ("empty ground-truth range", lambda c: c.gts["len"].__setitem__(0, 0)),
    ("negative ground-truth range", lambda c: c.gts["len"].__setitem__(0, -4096)),
    ("kernel index past the names", lambda c: c.cmds["kernel"].__setitem__(0, len(c.names))),
    ("bad kind", lambda c: c.cmds["kind"].__setitem__(0, 7)),
])
def test_loader_rejects_out_of_range_tables(tmp_path, name, mutate):
    _corrupt(tmp_path, mutate)
