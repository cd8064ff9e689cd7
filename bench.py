#!/usr/bin/env python
"""Decode-step benchmark (BASELINE.json metric: batch-1 decode ms/token and HBM
GB/s vs the roofline, Llama-3.1-8B bf16, 4k-token KV cache).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one decode step (one token per batch row) of the whole model at a
fixed context: every step reads all weights and the 4096(+1)-position KV
cache.  Weights are synthetic (device-side seeded init of the Llama-3.1-8B
shape; no checkpoint, no network).  Inputs (15.5 GB) are far larger than the
126 MB L2, so no flush is needed between steps.

Printed on rank 0 as ONE JSON line.  `value` = device time per token (CUDA
events on the launching stream, inputs resident in HBM); `e2e` = the same
metric through the public C-ABI call with host token input and host logits
output (H2D + D2H inside the timed region).

N > 1 GPUs (`--gpus N`; launched under torchrun by the driver, or re-executed
under torch.distributed.run by this script): the model is tensor-parallel
sharded over the N ranks (head-split attention, column /
row-split projections, vocabulary-split LM head), one process per GPU, the two
per-layer residual exchanges and the argmax exchange done inside the
persistent kernel over CUDA-IPC-mapped peer memory (NVLink P2P).  Total work
is fixed ("scaling": "strong", N = 1 included: it is the same model on one
GPU); `value` = the max over ranks of the device time per token.
`--replicas` runs N independent whole-model replicas instead ("weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode_ms_per_token"
UNIT = "ms/token"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama31_8b")
    ap.add_argument("--ctx", type=int, default=4096)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--quant", type=int, default=0, choices=[0, 4, 8],
                    help="weight-only quantization bits (BASELINE config Q)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent whole-model replicas instead of TP-N shards")
    ap.add_argument("--mode", default="fused_overlap",
                    choices=["fused_overlap", "fused", "baseline"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--calibrate", type=int, default=8,
                    help="ffb_calibrate iterations before timing (0 = uniform plan)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(cfg, ctx: int) -> int:
    """streamed weights (StoreLayout::streamed_weight_bytes,
    tensor_store.hpp:170-174) + KV read incl. the current token + embedding
    rows + f32 norm gains."""
    kv = cfg.batch * cfg.layers * cfg.n_kv_heads * 2 * cfg.d_head * 2 * (ctx + 1)
    return (cfg.streamed_weight_bytes() + kv + cfg.batch * cfg.d_model * 2 +
            (2 * cfg.layers + 1) * cfg.d_model * 4)


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(model: str, batch: int, ctx: int, quant: int = 0):
    """dram bytes per launch of the decode kernel from the committed ncu
    --set full summary (profiles/) of the same model / batch / context /
    weight format, or None."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_*.json"))):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        if (d.get("model") == model and d.get("batch") == batch and d.get("ctx") == ctx
                and int(d.get("quant", 0)) == quant):
            best = d.get("dram_bytes_per_launch")
    return best


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU side
def bench_config(args, tp: int, world: int) -> dict:
    """The `config` object both arms print (same workload wording)."""
    q = f"int{args.quant}" if args.quant else "bf16"
    return {
        "workload": f"{args.model} {q} decode step, batch {args.batch}, {args.ctx}-token KV cache"
                    + (f", tensor-parallel {tp}" if tp > 1 else ""),
        "model": args.model, "global_batch": args.batch * (world // tp), "seq_len": args.ctx,
        "parallelism": (f"tp{tp}" if tp > 1 else f"replicas{world}") if world > 1 else "single",
        "mode": args.mode,
        "l2": "weights + KV streamed per step exceed the 126 MB L2 (no flush needed)",
    }


def cpu_reference_ms_per_token(model: str, ctx: int, batch: int, quant: int, steps: int,
                               budget_s: float):
    """Times the reference's own CPU decode step (fusesim::reference_forward,
    reference.hpp:37-139, compiled unchanged into oracle/_ref; single-threaded
    like the reference) at FULL depth and width: the whole model, full
    vocabulary, a `ctx`-position cache, median of up to `steps` steps (fewer
    when they would exceed `budget_s`; the count is reported).  Weights are
    shape-correct deterministic values (ref_init_fast: the f64 arithmetic does
    not depend on them).  Falls back to the C restatement (kind "port",
    oracle/liboracle.so) when the reference build is absent."""
    import oracle as O
    from paper_2505_22758_b200 import model_preset
    cfg = model_preset(model)
    kind = "reference" if O.ref_available() else "port"
    oc = O.ModelCfg(cfg.layers, cfg.d_model, cfg.d_inter, cfg.d_head, cfg.n_q_heads,
                    cfg.n_kv_heads, cfg.vocab_size, batch=batch,
                    quant_bits=4 if quant == 4 else 0)
    t0 = time.perf_counter()
    if kind == "reference":
        st = O.RefStore(oc, None, ctx + 2)
    else:
        st = O.OracleStore(oc, 1234, ctx + 2, nthreads=1)
    init_s = time.perf_counter() - t0
    toks = [17 + b for b in range(batch)]

    def one():
        if kind == "reference":
            return st.time_forward(toks, ctx, 1)
        for l in range(oc.layers):
            st.set_length(l, ctx)
        t = time.perf_counter()
        st.forward(toks, ctx)
        return time.perf_counter() - t

    ts = [one()]
    n = max(1, min(steps, int(budget_s / max(ts[0], 1e-6))))
    while len(ts) < n:
        ts.append(one())
    st.close()
    med = statistics.median(ts)
    return {
        "value": med * 1e3 / batch,
        "unit": UNIT,
        "cores": 1,
        "kind": kind,
        "steps_timed": len(ts),
        "sample": (f"reference_forward (f64, single-threaded, as shipped) on the full {model} "
                   f"({oc.layers} layers, d_model {oc.d_model}, vocab {oc.vocab_size}), batch "
                   f"{batch}, ctx {ctx}: median of {len(ts)} step(s) of {steps} requested "
                   f"({min(ts):.2f}-{max(ts):.2f} s each; store init {init_s:.1f} s untimed)"
                   + ("; int8 is not in the reference: bf16 weights timed" if quant == 8 else "")),
        "host_cores_available": os.cpu_count(),
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # the CPU reference runs once, on rank 0
    tp = world if (world > 1 and not args.replicas) else 1
    base = cpu_reference_ms_per_token(args.model, args.ctx, args.batch, args.quant, args.steps,
                                      budget_s=180.0)
    v = base["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": base["steps_timed"], "warmup": 0,
        "ms_per_step": round(v * args.batch, 3), "higher_is_better": False,
        "scaling": "weak" if args.replicas else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (shape-correct deterministic weights; values do not affect timing)",
        "config": bench_config(args, tp, world),
        "cpu_baseline": base,
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU side
def run_ours(args):
    import numpy as np
    import torch
    from paper_2505_22758_b200 import DecodeModel, RunMode, model_preset

    rank, world, local = dist_env()
    n_dev = max(1, torch.cuda.device_count())
    # one rank per GPU; more ranks than GPUs (a functional check of the N > 1
    # path on one GPU, under MPS) share devices: SMs split between the
    # co-resident persistent kernels and host plumbing over gloo (NCCL
    # refuses two ranks on one device).  Timings of a shared GPU are not
    # per-GPU numbers and are flagged in the line.
    share = world > n_dev
    dev = local % n_dev
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if share else "nccl")
    grid = 0
    if share:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        grid = sms // -(-world // n_dev)
    cfg = model_preset(args.model).replace(batch=args.batch, quant_bits=args.quant)
    ctx = args.ctx
    tp = world if (world > 1 and not args.replicas) else 1
    mode = {"fused_overlap": RunMode.FUSED_OVERLAP, "fused": RunMode.FUSED,
            "baseline": RunMode.BASELINE}[args.mode]
    m = DecodeModel(cfg, ctx + 8, device=dev, mode=mode, tp_rank=rank if tp > 1 else 0,
                    tp_size=tp, grid=grid)
    # the in-kernel exchange stores into peer GPUs' memory (NVLink P2P); a box
    # without P2P between the group's GPUs runs the host-NCCL multi-kernel
    # TP path instead (RunMode.BASELINE_NCCL), flagged in the line
    p2p_ok = share or tp == 1 or all(torch.cuda.can_device_access_peer(dev, j)
                                     for j in range(min(world, n_dev)) if j != dev)
    if tp > 1 and world > 1:
        import torch.distributed as dist
        flag = torch.tensor([1 if p2p_ok else 0], dtype=torch.int32,
                            device="cpu" if share else f"cuda:{dev}")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        p2p_ok = bool(flag.item())
    if tp > 1 and p2p_ok:  # wire the TP group: all-gather every rank's exchange-buffer blob
        from paper_2505_22758_b200 import all_gather_tp_blobs
        m.tp_connect(all_gather_tp_blobs(m.tp_blob()))
    elif tp > 1:
        from paper_2505_22758_b200 import broadcast_nccl_id
        m.tp_nccl_init(broadcast_nccl_id())
        mode = RunMode.BASELINE_NCCL
        m.set_mode(mode)
    m.init_synthetic(1234)
    if args.calibrate and tp == 1 and not share:  # per-SM load balance (setup, outside the timed region)
        for l in range(cfg.layers):
            m.set_length(l, ctx)
        m.calibrate(args.calibrate)
    info = m.info()
    stream = torch.cuda.Stream(device=dev)
    tokens = torch.arange(17, 17 + args.batch, dtype=torch.int64, device=f"cuda:{dev}")

    def reset():
        for l in range(cfg.layers):
            m.set_length(l, ctx)

    def device_loop(n, run_mode):
        m.set_mode(run_mode)
        for _ in range(n):
            reset()
            m.step_device(tokens.data_ptr(), ctx, 0, 0, stream.cuda_stream)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def timed(run_mode, k):
        device_loop(args.warmup, run_mode)
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        device_loop(k, run_mode)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return e0.elapsed_time(e1) / k

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- headline: device-resident inputs, K timed steps
    with ClockSampler(dev) as clk:
        ms = timed(mode, args.steps)
    ms = max_over_ranks(ms)

    # ---- e2e through the public C-ABI call: host tokens in, host logits out
    m.set_mode(mode)
    tok_host = np.arange(17, 17 + args.batch, dtype=np.int64)
    logits_host = torch.empty((cfg.batch, cfg.vocab_size), dtype=torch.float32,
                              pin_memory=True).numpy()
    greedy_host = torch.empty(cfg.batch, dtype=torch.int64, pin_memory=True).numpy()
    for _ in range(args.warmup):
        reset()
        m.step(tok_host, ctx, out=logits_host, greedy=greedy_host, stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        reset()
        m.step(tok_host, ctx, out=logits_host, greedy=greedy_host, stream=stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)

    # ---- the same kernels launched as a multi-kernel pipeline (fusion gain)
    variants = {}
    if not args.no_variants:
        for name, rm in (("baseline", RunMode.BASELINE), ("fused", RunMode.FUSED),
                         ("fused_overlap", RunMode.FUSED_OVERLAP)):
            if tp > 1 and not p2p_ok:  # these exchange in-kernel over peer memory
                break
            k = max(10, args.steps // 4)
            variants[name + "_ms_per_step"] = round(max_over_ranks(timed(rm, k)), 5)
        if tp > 1 and not share and torch.cuda.device_count() >= tp:
            if p2p_ok:  # (else already initialised as the main mode)
                from paper_2505_22758_b200 import broadcast_nccl_id
                m.tp_nccl_init(broadcast_nccl_id())
            # the host-NCCL multi-kernel baseline: the same
            # per-stage launches, residual sums as ncclAllReduce between them
            k = max(10, args.steps // 4)
            variants["baseline_nccl_ms_per_step"] = round(
                max_over_ranks(timed(RunMode.BASELINE_NCCL, k)), 5)
        m.set_mode(mode)
        # device-resident greedy generation (ffb_decode_loop): 32 tokens per
        # call, no host round trip between tokens; cache reset per call
        n_gen = 32
        start = torch.full((cfg.batch,), 17, dtype=torch.int64, device=f"cuda:{dev}")
        gen = torch.empty((n_gen, cfg.batch), dtype=torch.int64, device=f"cuda:{dev}")

        def gen_loop(k):
            for _ in range(k):
                for l in range(cfg.layers):  # generation starts n_gen positions back
                    m.set_length(l, ctx - n_gen)
                m.decode_loop(start.data_ptr(), ctx - n_gen, n_gen, gen.data_ptr(), False,
                              stream.cuda_stream)
        torch.cuda.synchronize(dev)  # start / gen were written on the default stream
        gen_loop(2)
        torch.cuda.synchronize(dev)
        barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        k = max(2, args.steps // 32)
        g0.record(stream)
        gen_loop(k)
        g1.record(stream)
        torch.cuda.synchronize(dev)
        variants["decode_loop_ms_per_token"] = round(
            max_over_ranks(g0.elapsed_time(g1) / (k * n_gen)) / cfg.batch, 5)
        if tp == 1:
            # prompt ingestion as GEMMs (ffb_prefill): a 512-token
            # prompt (per batch row) ending at the bench context, host wall
            # clock around the synchronous call (prompt copy and last logits
            # included), best of 3 after one warm-up
            import time as _time
            n_pf = min(512, 1024 // cfg.batch, ctx)
            prompt = np.random.default_rng(3).integers(0, cfg.vocab_size, size=(n_pf, cfg.batch))
            best = float("inf")
            for r in range(4):
                for l in range(cfg.layers):
                    m.set_length(l, ctx - n_pf)
                t0 = _time.perf_counter()
                m.prefill(prompt, ctx - n_pf, logits=False)
                if r:
                    best = min(best, _time.perf_counter() - t0)
            variants["prefill_prompt_tokens"] = int(n_pf * cfg.batch)
            variants["prefill_ms"] = round(best * 1e3, 3)
            variants["prefill_tokens_per_s"] = round(n_pf * cfg.batch / best, 1)
            for l in range(cfg.layers):
                m.set_length(l, ctx)

    algo = algorithmic_bytes(cfg, ctx)
    peak, peak_kind = measured_peak()
    # per GPU: a TP rank streams 1/tp of the model (its shard); the roofline
    # is per device either way
    achieved = algo / tp / (ms * 1e-3) / 1e9
    launches = info["launches_per_step"] if mode != RunMode.BASELINE else cfg.layers * 5 + 1

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:  # bounded sample: ~2 full-depth steps (about 10-30 s of CPU work)
            cpu = cpu_reference_ms_per_token(args.model, ctx, args.batch, args.quant, 2,
                                             budget_s=20.0)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms / args.batch, 5), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": False,
            "scaling": "weak" if args.replicas else "strong", "vs_baseline": None,
            "n_ranks_tp": tp,
            **({"tp_exchange": ("in-kernel over CUDA-IPC memory on the shared GPU" if share
                                else "in-kernel over NVLink peer memory") if p2p_ok
                else "host NCCL between per-stage launches (no P2P between the GPUs)"} if tp > 1 else {}),
            **({"shared_gpu": f"{world} ranks on {n_dev} GPU(s): functional check, not a "
                              f"per-GPU timing"} if share else {}),
            "dtype": f"int{args.quant} weights, f32 math" if args.quant else "bf16",
            "data": "synthetic (seeded device-side init of the model shape)",
            "config": bench_config(args, tp, world),
            "tokens_per_s": round(1e3 * args.batch * (world // tp) / ms, 2),
            "roofline": {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                "frac_of_8TBs": round(achieved / 8000.0, 4),
                "algorithmic_bytes_per_launch": algo // tp,
                "traffic": ncu_traffic(args.model, args.batch, ctx, args.quant) if tp == 1 else None,
                "kernel": "ffb200::decode_step_kernel (1 persistent launch per step)",
            },
            "e2e": {"value": round(e2e_ms / args.batch, 5), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * cfg.batch,
                    "d2h_bytes_per_step": 4 * cfg.batch * cfg.vocab_size // tp + 8 * (cfg.batch + 1)},
            "gpu_launches": launches * args.steps,
            "variants": variants,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "kernel_info": info,
            "plan": {"calibrate_iterations": args.calibrate,
                     "sm_weight_min": round(float(m.plan_weights().min()), 4),
                     "sm_weight_max": round(float(m.plan_weights().max()), 4)},
        }
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torchrun (the driver does this itself)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)]
        os.execv(sys.executable, cmd + sys.argv[1:])
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
