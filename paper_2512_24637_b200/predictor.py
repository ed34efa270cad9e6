"""Drop-in working-set predictor API (reference predictor.py:18-87), with the
evaluation on the GPU (csrc/k_predict.cu).

`predict`, `predict_allocation` and `ground_truth_prediction` keep the
reference signatures; each call runs the device predictor on a one-command
batch.  `predict_task` is the batched form the engine itself uses.

The per-call path reuses one predictor context per (page size, mode, device)
-- each call registers its commands as a fresh task of that context, and
the context is recycled every `_RECYCLE` calls -- so a call costs the K1
launches and their round trips, not a context's creation and teardown.
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


_RECYCLE = 1024
_CTX: dict = {}


def _context(page_size: int, pred: int, device: int):
    """(context, fresh task index) from the per-(page, mode, device) cache."""
    key = (page_size, pred, device)
    ent = _CTX.get(key)
    if ent is None or ent[1] >= _RECYCLE:
        if ent is not None:
            ent[0].close()
        ctx = _abi.Context(page_size, 1, predictor=pred, device=device, flags=_abi.F_LOOSE_DOMAIN)
        ctx.set_domain([(0, 1)])
        ent = _CTX[key] = [ctx, 0]
    ent[1] += 1
    return ent[0], ent[1] - 1


def predict_task(commands, page_size: int, mode: str = "template", descriptors: dict | None = None,
                 allocations: Sequence = (), device: int = 0) -> list:
    """Predict every command on the device; returns [Prediction]."""
    pred = {"template": _abi.PRED_TEMPLATE, "allocation": _abi.PRED_ALLOCATION,
            "oracle": _abi.PRED_TRUTH}[mode]
    commands = list(commands)
    ctx, ti = _context(page_size, pred, device)
    ctx.add_task(ti, [(a.base_addr, a.size_bytes) for a in allocations])
    kid, lossy = {}, []
    if pred == _abi.PRED_TEMPLATE and descriptors:
        names, rules, offs, lossy = _abi.lower_rules(descriptors)
        kid = {n: k for k, n in enumerate(names)}
        ctx.set_rules(ti, rules, offs)
    comp = ctx.add_commands(ti, _abi.encode_commands(commands, kid))
    out = []
    for i, c in enumerate(commands):
        k = kid.get(c.kernel_name, -1)
        ok = bool(comp[i]) and not (c.kind is CommandKind.KERNEL and k >= 0 and lossy[k])
        out.append(Prediction(PageSet._raw(ctx.read_pages(ti, i, 0)), ok))
    return out


def predict(descriptors: dict, cmd, page_size: int) -> Prediction:
    # only the command's own kernel descriptor is lowered (predictor.py:31-33
    # reads no other)
    d = descriptors.get(cmd.kernel_name) if getattr(cmd.kind, "value", cmd.kind) == "KERNEL" else None
    return predict_task([cmd], page_size, "template", {cmd.kernel_name: d} if d is not None else {})[0]


def predict_allocation(allocations, cmd, page_size: int) -> Prediction:
    return predict_task([cmd], page_size, "allocation", allocations=allocations)[0]


def ground_truth_prediction(cmd, page_size: int) -> Prediction:
    return predict_task([cmd], page_size, "oracle")[0]


def accuracy(predicted: PageSet, actual: PageSet) -> tuple:
    """(F-, F+) over |actual| as the reference computes it (predictor.py:80-87)."""
    n = len(actual)
    if n == 0:
        return (0.0, 0.0)
    return (len(actual - predicted) / n, len(predicted - actual) / n)
