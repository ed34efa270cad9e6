"""The C ABI (include/msched_b200.h) without a GPU: the library loads,
exports every declared entry point, and the ctypes/numpy mirrors have the
header's exact struct layouts (checked against gcc's sizeof/offsetof)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2512_24637_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msched_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(msg_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing
    assert set(names) == set(_abi.EXPORTS)


def _c_layout(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "msched_b200.h"
#define S(t) printf(#t " %zu\\n", sizeof(t));
#define O(t, f) printf(#t "." #f " %zu\\n", offsetof(t, f));
int main(void) {
  S(msg_cfg) S(msg_arg) S(msg_cmd) S(msg_range) S(msg_expr) S(msg_rule) S(msg_window)
  S(msg_switch_out) S(msg_touch_out) S(msg_stats)
  O(msg_cmd, dims) O(msg_cmd, dev_addr) O(msg_rule, e) O(msg_expr, slot) O(msg_arg, raw_off)
  O(msg_switch_out, first_missing_pages) O(msg_touch_out, next_missing_pages) O(msg_stats, ms_bytes)
  O(msg_cfg, flags) O(msg_stats, run_ms) O(msg_stats, ms_dev_ms) O(msg_stats, ms_ev_passes)
  return 0;
}
""")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    return dict(line.rsplit(" ", 1) for line in out.strip().splitlines())


def test_struct_layouts_match_header(tmp_path):
    c = {k: int(v) for k, v in _c_layout(tmp_path).items()}
    assert c["msg_cfg"] == ctypes.sizeof(_abi.Cfg)
    assert c["msg_cfg.flags"] == _abi.Cfg.flags.offset
    assert c["msg_arg"] == _abi.ARG_DT.itemsize and c["msg_arg.raw_off"] == _abi.ARG_DT.fields["raw_off"][1]
    assert c["msg_cmd"] == _abi.CMD_DT.itemsize
    assert c["msg_cmd.dims"] == _abi.CMD_DT.fields["dims"][1]
    assert c["msg_cmd.dev_addr"] == _abi.CMD_DT.fields["dev_addr"][1]
    assert c["msg_range"] == _abi.RANGE_DT.itemsize
    assert c["msg_expr"] == _abi.EXPR_DT.itemsize and c["msg_expr.slot"] == _abi.EXPR_DT.fields["slot"][1]
    assert c["msg_rule"] == _abi.RULE_DT.itemsize and c["msg_rule.e"] == _abi.RULE_DT.fields["e"][1]
    assert c["msg_window"] == ctypes.sizeof(_abi.Window)
    assert c["msg_switch_out"] == ctypes.sizeof(_abi.SwitchOut)
    assert c["msg_switch_out.first_missing_pages"] == _abi.SwitchOut.first_missing_pages.offset
    assert c["msg_touch_out"] == ctypes.sizeof(_abi.TouchOut)
    assert c["msg_touch_out.next_missing_pages"] == _abi.TouchOut.next_missing_pages.offset
    assert c["msg_stats"] == ctypes.sizeof(_abi.Stats) and c["msg_stats.ms_bytes"] == _abi.Stats.ms_bytes.offset
    assert c["msg_stats.run_ms"] == _abi.Stats.run_ms.offset
    assert c["msg_stats.ms_dev_ms"] == _abi.Stats.ms_dev_ms.offset
    assert c["msg_stats.ms_ev_passes"] == _abi.Stats.ms_ev_passes.offset


def test_slot_codes_and_rule_lowering():
    assert _abi.slot_code("gx") == 2 and _abi.slot_code("bz") == 2 | (5 << 2)
    assert _abi.slot_code("a3") == 3 << 2
    code = _abi.slot_code("a1+8w64")
    assert code & 3 == 1 and (code >> 2) & 0xFFFF == 1 and (code >> 18) & 0xFFFFFFFF == 8 and (code >> 50) & 1
    from paper_2512_24637_b200.workload import gen_template_corpus
    from paper_2512_24637_b200.analyzer import build_descriptors

    names, rules, offs, lossy = _abi.lower_rules(build_descriptors(gen_template_corpus(12, seed=1).task))
    assert len(names) == 12 and offs[-1] == len(rules) and len(lossy) == 12
    assert all(rules["e"][:, 0]["den"] > 0)


@pytest.mark.skipif(_abi.cuda_device_count() > 0, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_a_gpu():
    """The product path refuses to run without a GPU instead of silently
    falling back to host code."""
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _abi.Context(4096, 16)
