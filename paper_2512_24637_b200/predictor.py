"""Drop-in working-set predictor API (reference predictor.py:18-87), with the
evaluation on the GPU (csrc/k_predict.cu).

`predict`, `predict_allocation` and `ground_truth_prediction` keep the
reference signatures and run the device predictor on the one command.
`predict_task` is the batched form the engine itself uses: one upload, the
K1 launches, and one device-to-host copy of every command's runs.

The per-call path keeps one predictor context per (page size, mode,
device) and, in it, one task per kernel descriptor (template mode) or per
allocation table (allocation mode): a call appends its command to that
task -- the rules and allocations are lowered and uploaded once -- and
reads the command's runs back.  Contexts are recycled every `_RECYCLE`
commands.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from . import _abi
from .model import CommandKind, PageSet

__all__ = ["Prediction", "predict", "predict_allocation", "ground_truth_prediction", "predict_task", "accuracy"]


@dataclass
class Prediction:
    pages: PageSet
    complete: bool = True


_RECYCLE = 4096
_CTX: dict = {}
_PRED = {"template": _abi.PRED_TEMPLATE, "allocation": _abi.PRED_ALLOCATION, "oracle": _abi.PRED_TRUTH}


class _Slot:
    """One context of the per-call cache: its tasks by key."""

    def __init__(self, page_size, pred, device):
        self.ctx = _abi.Context(page_size, 1, predictor=pred, device=device, flags=_abi.F_LOOSE_DOMAIN)
        self.ctx.set_domain([(0, 1)])
        self.tasks = {}     # key -> [task index, commands so far, kernel ids, lossy flags, pinned objects]
        self.ntasks = 0
        self.ncmds = 0


def _slot(page_size: int, pred: int, device: int) -> _Slot:
    key = (page_size, pred, device)
    s = _CTX.get(key)
    if s is None or s.ncmds >= _RECYCLE:
        if s is not None:
            s.ctx.close()
        s = _CTX[key] = _Slot(page_size, pred, device)
    return s


def _task(s: _Slot, key, allocations=(), descriptors=None, pin=()):
    ent = s.tasks.get(key)
    if ent is None:
        ti = s.ntasks
        s.ntasks += 1
        s.ctx.add_task(ti, [(a.base_addr, a.size_bytes) for a in allocations])
        kid, lossy = {}, []
        if descriptors:
            names, rules, offs, lossy = _abi.lower_rules(descriptors)
            kid = {n: k for k, n in enumerate(names)}
            s.ctx.set_rules(ti, rules, offs)
        ent = s.tasks[key] = [ti, 0, kid, lossy, pin]
    return ent


def _one(s: _Slot, ent, cmd) -> Prediction:
    ti, n, kid, lossy = ent[0], ent[1], ent[2], ent[3]
    try:
        comp = s.ctx.add_commands(ti, _abi.encode_commands([cmd], kid))
    except Exception:
        # the task's tables may hold part of the failed command: later calls
        # start a fresh task for this key
        for k, v in list(s.tasks.items()):
            if v is ent:
                del s.tasks[k]
        raise
    ent[1] += 1
    s.ncmds += 1
    k = kid.get(cmd.kernel_name, -1)
    ok = bool(comp[0]) and not (cmd.kind is CommandKind.KERNEL and k >= 0 and lossy[k])
    return Prediction(PageSet._raw(s.ctx.read_pages(ti, n, 0)), ok)


def predict_task(commands, page_size: int, mode: str = "template", descriptors: dict | None = None,
                 allocations: Sequence = (), device: int = 0) -> list:
    """Predict every command on the device; returns [Prediction]."""
    pred = _PRED[mode]
    commands = list(commands)
    s = _slot(page_size, pred, device)
    ti = s.ntasks          # a fresh task for the batch
    s.ntasks += 1
    s.ncmds += len(commands)
    s.ctx.add_task(ti, [(a.base_addr, a.size_bytes) for a in allocations])
    kid, lossy = {}, []
    if pred == _abi.PRED_TEMPLATE and descriptors:
        names, rules, offs, lossy = _abi.lower_rules(descriptors)
        kid = {n: k for k, n in enumerate(names)}
        s.ctx.set_rules(ti, rules, offs)
    comp = s.ctx.add_commands(ti, _abi.encode_commands(commands, kid))
    out = []
    if not commands:
        return out
    runs, off = s.ctx.read_pages_range(ti, 0, len(commands), 0)   # one copy for the batch
    rl = runs.tolist()
    for i, c in enumerate(commands):
        k = kid.get(c.kernel_name, -1)
        ok = bool(comp[i]) and not (c.kind is CommandKind.KERNEL and k >= 0 and lossy[k])
        out.append(Prediction(PageSet._raw([tuple(r) for r in rl[off[i]:off[i + 1]]]), ok))
    return out


def predict(descriptors: dict, cmd, page_size: int) -> Prediction:
    # only the command's own kernel descriptor is lowered (predictor.py:31-33
    # reads no other); its task in the cached context is keyed by the
    # descriptor object (kept alive by the cache, so the id is not reused)
    d = descriptors.get(cmd.kernel_name) if getattr(cmd.kind, "value", cmd.kind) == "KERNEL" else None
    s = _slot(page_size, _abi.PRED_TEMPLATE, 0)
    ent = _task(s, ("t", cmd.kernel_name, id(d)), descriptors={cmd.kernel_name: d} if d is not None else None,
                pin=(d,))
    return _one(s, ent, cmd)


def predict_allocation(allocations, cmd, page_size: int) -> Prediction:
    allocations = list(allocations)
    s = _slot(page_size, _abi.PRED_ALLOCATION, 0)
    ent = _task(s, ("a", tuple((a.base_addr, a.size_bytes) for a in allocations)), allocations=allocations)
    return _one(s, ent, cmd)


def ground_truth_prediction(cmd, page_size: int) -> Prediction:
    s = _slot(page_size, _abi.PRED_TRUTH, 0)
    return _one(s, _task(s, ("g",)), cmd)


def accuracy(predicted: PageSet, actual: PageSet) -> tuple:
    """(F-, F+) over |actual| as the reference computes it (predictor.py:80-87)."""
    n = len(actual)
    if n == 0:
        return (0.0, 0.0)
    return (len(actual - predicted) / n, len(predicted - actual) / n)
