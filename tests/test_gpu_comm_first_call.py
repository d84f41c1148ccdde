"""Regression: a process whose FIRST call of the stage carries a communicator
(bench.py at N > 1, or --force-comm) must not deadlock.  The comm stream's
spinning wait kernels are resident while the main stream launches the step;
under CUDA's lazy module loading a kernel's first launch could wait for the
device to go idle.  The library now runs a path's first call once without the
communicator (attn_softmax_fwd_bwd_ex).  Lazy loading is per process, so the
check runs in a fresh subprocess with CUDA_MODULE_LOADING=LAZY."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs
cfg = CONFIGS[{name!r}]
inp = make_inputs(cfg)
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
        dv["W_out"], 1.0 / global_valid_tokens(cfg, cfg.B))
comm = binding.attn_comm_init(binding.attn_comm_get_unique_id(), 1, 0, 0)
out = st(*args, comm=comm)              # the process's first call carries the communicator
for _ in range(3):
    st(*args, out=out, comm=comm)
binding.attn_comm_poll(comm, 60000)
torch.cuda.synchronize()
ref = st(*args)
torch.cuda.synchronize()
assert all(torch.equal(out[k], ref[k]) for k in ("loss", "dW_out", "dW_c", "dH_dec", "dH_enc"))
binding.attn_comm_destroy(comm)
print("ok")
"""


@pytest.mark.parametrize("name", ["small", "paper"])
def test_first_call_with_communicator(cuda_lib, name):
    env = dict(os.environ, CUDA_MODULE_LOADING="LAZY")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, name=name)], env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
