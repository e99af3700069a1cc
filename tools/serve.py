"""Wall-clock serving sweep on one B200: QLLM vs FCFS on the paper workload (one JSON per rate and
seed), with the SM clocks sampled over each rate's runs (nvidia-smi, as in bench.py)."""
import argparse, json, sys, time
from dataclasses import replace
sys.path.insert(0, ".")
import torch
from bench import ClockSampler
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel
from paper_2503_09304_b200.serving import compare, warm_up


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral", choices=["mixtral", "qwen"])
    ap.add_argument("--rates", default="7")
    ap.add_argument("--seeds", default="0")
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--schedulers", default="baseline,qllm")
    ap.add_argument("--mbs", type=int, default=32)
    ap.add_argument("--slo-ms", type=float, default=3000.0)
    ap.add_argument("--layers", type=int, default=0, help="debug only: fewer layers")
    ap.add_argument("--kv-gib", type=float, default=0.0,
                    help="KV admission capacity in GiB (default: the reference's 8 GiB ledger)")
    ap.add_argument("--keep-engine", action="store_true", help="keep the engine stats in the output")
    args = ap.parse_args()
    cfg = MIXTRAL_8X7B if args.model == "mixtral" else QWEN15_MOE_A27B
    if args.layers:
        cfg = replace(cfg, num_layers=args.layers)
    t = time.perf_counter()
    model = DecoderMoEModel(cfg)
    torch.cuda.synchronize()
    print(json.dumps({"init_s": time.perf_counter() - t, "model": cfg.name,
                      "mem_gb": torch.cuda.memory_allocated() / 1e9}), flush=True)
    warm_up(model, args.mbs)
    for rate in [float(r) for r in args.rates.split(",")]:
        for seed in [int(s) for s in args.seeds.split(",")]:
            sampler = ClockSampler(torch.cuda.current_device())
            out = compare(model, rate, args.duration, seed=seed, max_batch_size=args.mbs, slo_ms=args.slo_ms,
                          schedulers=args.schedulers.split(","),
                          kv_capacity_bytes=args.kv_gib * 1024**3 if args.kv_gib else None)
            out["clocks"] = sampler.stop()
            out["model"] = cfg.name
            out["seed"] = seed
            if not args.keep_engine:
                for k in ("fcfs", "qllm", "never-preempt"):
                    if k in out:
                        out[k].pop("engine", None)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
