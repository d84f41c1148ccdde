python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_lstm.py -q -x 2>&1 | tail -4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 6 --csv python scripts/decode_profile.py 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5, $(NF)}' | cut -c1-120
python - <<'PY'
import sys, os
sys.path.insert(0, ".")
from dataclasses import replace
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import DecodeStep, to_device
from synthetic import CONFIGS, make_inputs
cfg = replace(CONFIGS["paper"], N=5, lengths="full")
inp = make_inputs(cfg)
dv = to_device(inp, cfg.dtype)
step = DecodeStep(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, 5)
for thr in (0, 1, 0, 1):
    binding.attn_softmax_set_option("decode_thr", thr)
    for _ in range(3): step(dv["H_dec"], dv["H_enc"], inp["src_len"], dv["W_c"], dv["W_out"])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): step(dv["H_dec"], dv["H_enc"], inp["src_len"], dv["W_c"], dv["W_out"])
    b.record(); torch.cuda.synchronize()
    print("decode_thr", thr, a.elapsed_time(b) / 20 * 1e3, "us")
PY
