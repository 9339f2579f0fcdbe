"""ncu target: two quantizer rounds of a 2-layer DeepSeek-shape model with the B operands fused (flux_quantize_weights_bops)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import torch  # noqa: E402
from paper_2508_19078_b200 import synthetic
from paper_2508_19078_b200.driver import ModelShape, QuantizedModel
cfg = synth.CONFIGS["deepseek_moe"].with_(n_layers=2)
shape = ModelShape.of(cfg)
m = synthetic.master_weights(cfg)
qm = QuantizedModel(shape, with_bops=True)
for _ in range(2):
    qm.quantize_from(m)
torch.cuda.synchronize()
print("ok")
