import sys, ctypes as C
sys.path.insert(0, ".")
from paper_2512_24637_b200 import _abi
_abi.LIB_PATH = "tools/libmsched_fwts.so"
from paper_2512_24637_b200 import engine, scenarios
from paper_2512_24637_b200.analyzer import build_descriptors
tasks, hw, pol = scenarios.config2_llama8b()
descs = {t.id: build_descriptors(t) for t in tasks}
sim = engine.Simulator(tasks, hw, pol, engine.Mode.proactive(), descriptors=descs)
for r in range(2):
    sim.reset(); sim.run(); sim.ctx.sync()
lib = _abi.load()
out = (C.c_ulonglong * 32)()
lib.msg_dbg_fw_ts(out)
n = out[0]
prev = 0
print("launches", n)
for i in range(1, 11):
    v = out[i] / n / 1e3
    print(f"T{i}: {v:7.2f} us (+{v - prev:5.2f})")
    prev = v
