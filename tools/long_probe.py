"""Sustained single-gate probe: one k = 6 Haar gate 300 times on a 34q state
(dense random state, or `basis` for |0>), per-20-pass mean times."""
import sys, json, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2111_06868_b200 as hq
from hq_inputs import haar_sweep_gate
n = 34
from hq_inputs.states import random_state_torch
dense = len(sys.argv) < 2 or sys.argv[1] != "basis"
psi_t = random_state_torch(n, "cuda", seed=32)
st = torch.cuda.Stream()
torch.cuda.synchronize()
s = hq.hq_state_create_from_buffers(n, "c64", psi_t.data_ptr(), st.cuda_stream)
if not dense:
    hq.hq_state_init_basis(s, 0)      # the sparse |0>-derived comparison
g = haar_sweep_gate(n, 6, "b:16-17-18-22-23-24", seed=7)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
t0 = time.time()
for e0, e1 in ev:
    e0.record(st); hq.hq_apply_matrix(s, g.U, g.qubits); e1.record(st)
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in ev]
for i in range(0, 300, 20):
    print(i, round(sum(ms[i:i+20]) / 20, 2))
