import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1809_02697_b200 import DeviceProgram, ExecutablePlan, ScheduleDb, build_model, compile_graph, model_input
from paper_1809_02697_b200.tuning import DEFAULT_DB
from paper_1809_02697_b200.timing import graph_time
g = build_model("resnet50", batch=64)
prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16", db=ScheduleDb(DEFAULT_DB))), 0, "bf16")
prog.set_inputs(model_input(g))
flush = torch.empty(64 * 1024 * 1024, device="cuda")
f = lambda: flush.zero_()
hs = [i for i, n in enumerate(prog.launch_names) if n.startswith("head")]
full = min(graph_time(prog, lambda i: True, 20, f) for _ in range(3))
nohead = min(graph_time(prog, lambda i: i not in hs, 20, f) for _ in range(3))
print(f"COOP={os.environ.get('NEOB200_HEAD_COOP', '1')}: step {full*1e3:.4f} ms, without head {nohead*1e3:.4f} ms, head {1e6*(full-nohead):.1f} us")
