import cProfile, pstats, sys, io
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200.mixtral import QWEN15_MOE_A27B, MIXTRAL_8X7B, DecoderMoEModel
from paper_2503_09304_b200.serving import compare, warm_up
cfg = QWEN15_MOE_A27B if sys.argv[1] == "qwen" else MIXTRAL_8X7B
m = DecoderMoEModel(cfg)
warm_up(m)
pr = cProfile.Profile()
pr.enable()
out = compare(m, 7.0, 6.0, schedulers=("qllm",))
pr.disable()
print({k: v for k, v in out["qllm"].items() if k != "engine"})
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
