"""The native analyzer (msg_analyze, host C++ in the C-ABI library) against
this package's host analyzer, which tests/test_host_golden.py pins to the
reference: identical descriptors (rules, exact coefficients, latencies and
uncovered fractions, bit for bit) on every trace shape the repo produces."""

import random

import pytest

from paper_2512_24637_b200 import analyzer
from paper_2512_24637_b200.model import Arg, ByteRange, Command, CommandKind, Task
from paper_2512_24637_b200.presets import get_preset
from paper_2512_24637_b200.scenarios import config1_gemm, llm_scenario, streaming_scenario
from paper_2512_24637_b200.workload import gen_template_corpus
from paper_2512_24637_b200.workload_extra import config3_mixed
from tests.golden import loader

HW = get_preset("rtx5080").with_capacity(96 << 20)


def _same(task):
    a = analyzer.build_descriptors(task, native=True)
    b = analyzer.build_descriptors(task, native=False)
    assert list(a) == list(b)
    assert analyzer.format_descriptors(a) == analyzer.format_descriptors(b)
    for k in a:
        assert a[k] == b[k], k


def test_generated_traces():
    tasks = list(llm_scenario(HW, 2.0, n_tasks=2, layers=4, decode_steps=3)[0])
    tasks += list(streaming_scenario(HW, 2.0, indirect_rate=0.01, seed=1)[0])
    tasks += list(config1_gemm()[0])
    tasks += list(config3_mixed(hbm_bytes=1 << 30, ratio=2.0, page_size=4096, task_offset=0,
                                timeslice_s=5e-4)[0])
    for t in tasks:
        _same(t)


@pytest.mark.parametrize("seed", range(6))
def test_planted_rule_corpora(seed):
    _same(gen_template_corpus(40, seed=seed).task)


def test_golden_traces():
    n = 0
    for case in loader.predictions():
        _same(loader.dec_task(case["task"]))
        n += 1
    assert n > 0


def test_fallback_paths_agree():
    """Arguments beyond 64 bits, ragged argument counts and zero-length
    regions go to the host path per kernel and still agree."""
    big = 1 << 70
    cmds = []
    for k in range(4):
        base = (1 << 40) + k * (1 << 20)
        cmds.append(Command(CommandKind.KERNEL, 1e-6, "wide", (Arg(base), Arg(big + k, 64), Arg(64 * (k + 1))),
                            ground_truth_access=(ByteRange(base, 64 * (k + 1)),)))
        cmds.append(Command(CommandKind.KERNEL, 1e-6, "ragged", (Arg(base),) + ((Arg(7),) if k % 2 else ()),
                            ground_truth_access=(ByteRange(base, 4096),)))
    _same(Task(id="edge", commands=cmds))


def test_random_linear_and_strided_kernels():
    rng = random.Random(9)
    cmds = []
    for rep in range(60):
        n, m = rng.randint(1, 400), rng.randint(1, 30)
        base = (1 << 40) + rep * (1 << 24)
        other = base + (1 << 22)
        ga = ByteRange(base, 8 * n * m)
        gb = tuple(ByteRange(other + j * 4 * n, 2 * n) for j in range(m))
        cmds.append(Command(CommandKind.KERNEL, 1e-6 * (1 + rep % 3), f"k{rep % 5}",
                            (Arg(base), Arg(other), Arg(n, 32), Arg(m, 32)), (max(1, n // 8), 1, 1), (m, 1, 1),
                            (ga,) + gb))
    _same(Task(id="rand", commands=cmds))


def test_binary_trace_columns(tmp_path):
    """Descriptors straight from MSIM-TRACE-BIN columns equal the host analyzer's."""
    from paper_2512_24637_b200 import tracebin

    tasks = list(llm_scenario(HW, 2.0, n_tasks=2, layers=4, decode_steps=3)[0])
    tasks.append(gen_template_corpus(30, seed=4).task)
    p = tmp_path / "t.msimb"
    tracebin.save_trace_bin(tasks, str(p))
    for orig, cols in zip(tasks, tracebin.load_trace_bin(str(p))):
        a = analyzer.build_descriptors(cols, native=True)
        b = analyzer.build_descriptors(orig, native=False)
        assert list(a) == list(b) and a == b
