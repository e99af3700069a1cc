import faulthandler, sys, time
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, ".")
import torch
from dataclasses import replace
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, DecoderMoEModel
from paper_2503_09304_b200.serving import serve_once
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate
m = DecoderMoEModel(replace(MIXTRAL_8X7B, num_layers=int(sys.argv[1]) if len(sys.argv) > 1 else 2))
tr = trace_for_rate(WorkloadSpec(duration_s=3.0, prompt_mean=64, output_mean=8), 4.0, seed=99)
t = time.time()
print(serve_once(m, tr, "qllm"), time.time() - t, flush=True)
