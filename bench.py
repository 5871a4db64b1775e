#!/usr/bin/env python3
"""bench.py -- ISRTF re-predict + select throughput on B200 (BASELINE.json metric).

One step = one scheduling iteration of ELIS Algorithm 1 lines 10-19: re-encode
every due request (prompt + partial response) with the BGE encoder, predict its remaining
tokens with the 8-FC head, and select the next batch (ISRTF, batch_cap).

Default workload = BASELINE.json configs[4] / the north_star (cfg5): BGE-base, 65,536
requests in flight; each iteration re-predicts the due set -- ceil(65,536 / 50) = 1,311 jobs
returning from a 50-token window -- into the in-flight table through out_slot, and
selects batch_cap 256 over all 65,536 cached keys.  With --gpus N (torchrun) the due set is
split at the quantiles of its encoder cost (elis_cost_split), each rank encodes its slice,
elis_predict_remaining_dist all-gathers the predictions into every rank's table (one fused
kernel over NVLink peer memory, or NCCL) and every rank runs the same select: strong scaling.
--workload cfg2 / cfg1 / cfg3 run the other BASELINE.json configs (full re-predict per step).

    python bench.py [--gpus N --steps K --warmup W] [--impl elis|reference] [--workload cfgX]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2505_09142_b200 import inputs  # noqa: E402

METRIC = "ISRTF re-predict+select predictions/sec and ms/iteration at 1/2/4/8 B200"
UNIT = "predictions/s"

# BASELINE.json configs as bench workloads.  cfg5 (the north_star target) is the default: BGE-base,
# 65,536 requests in flight, each scheduling iteration re-predicts the due set -- the jobs returning
# from a 50-token window, ceil(65,536 / 50) = 1,311 (Alg. 1 lines 10-18) --
# into the in-flight table and selects batch_cap 256 over every cached key (line 19).
WORKLOADS = {
    "cfg5": dict(config="base", inflight=65536, due=0, cap=256, lengths="trace", n=0),
    "cfg2": dict(config="base", inflight=0, due=0, cap=4, lengths="trace", n=256),
    "cfg1": dict(config="tiny", inflight=0, due=0, cap=4, lengths="fixed:64", n=16),
    "cfg3": dict(config="large", inflight=0, due=0, cap=4, lengths="uniform", n=4096),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["elis", "reference"], default="elis")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg5",
                    help="BASELINE.json config: cfg5 (default, north_star: 65,536 in flight, the due set "
                         "re-predicted, select over every cached key), cfg2 (256 requests fully re-predicted per "
                         "GPU), cfg1 (tiny), cfg3 (BGE-large, 4,096 uniform 32-512)")
    ap.add_argument("--config", choices=["tiny", "base", "large"], default=None, help="encoder (overrides the workload's)")
    ap.add_argument("--n", "--requests", dest="n", type=int, default=None,
                    help="batch workloads: requests re-predicted per GPU per step (--requests: the same, for torchrun "
                         "command lines, whose parser takes a bare --n for its own --nnodes / --nproc-per-node)")
    ap.add_argument("--total-requests", type=int, default=0,
                    help="batch workloads, strong scaling: this many requests per step in total, split evenly")
    ap.add_argument("--lengths", default=None, help="trace | uniform | fixed:L")
    ap.add_argument("--cap", type=int, default=None, help="batch_cap")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precision", choices=["bf16", "fp8", "fp16"], default=None,
                    help="encoder operands: default = the library default (elis.h ELIS_PREC_AUTO: fp16 for head dim "
                         "64, bf16 for the tiny d=32 encoder -- DESIGN.md R21), or bf16 / fp8 (row f4(i))")
    ap.add_argument("--residual", choices=["fp32", "fp16"], default=None,
                    help="residual stream: default = the library default (fp16 with fp16 operands, DESIGN.md R23)")
    ap.add_argument("--pooling", choices=["mean", "cls"], default="mean",
                    help="mean (P:359, default) or CLS (P:138) pooling (DESIGN.md R2)")
    ap.add_argument("--cls-last-layer", action="store_true",
                    help="with --pooling cls: the last layer computes only the CLS rows (SURVEY.md 8f row f4(ii))")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=12, help="requests in the oracle sample")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="N > 1 exchange -- peer: fused kernels storing into every rank's CUDA-IPC-mapped region "
                         "over NVLink (elis_peer_attach); nccl: ncclAllGather between kernels (elis_dist_attach)")
    ap.add_argument("--graph", choices=["on", "off"], default="on",
                    help="on: the timed steps replay CUDA graphs of the step's library calls (one per due window "
                         "for cfg5); the per-kernel breakdown and e2e stay eager")
    ap.add_argument("--inflight", type=int, default=None,
                    help="in-flight table slots (cfg5: 65,536); 0 = a batch workload")
    ap.add_argument("--due", type=int, default=None,
                    help="due requests per iteration over all GPUs (cfg5 default ceil(inflight / 50) = 1,311)")
    a = ap.parse_args(argv)
    preset = WORKLOADS[a.workload]
    due_given, n_given = a.due is not None, a.n is not None
    for k in ("config", "cap", "lengths", "n", "inflight", "due"):
        if getattr(a, k) is None:
            setattr(a, k, preset[k])
    if a.inflight > 0 and not due_given:
        # --requests with a table: due requests per GPU; else ceil(inflight / K) in total
        a.due = a.n * max(1, a.gpus) if n_given else -(-a.inflight // inputs.WINDOW_K)
    if a.inflight <= 0 and not a.n:
        a.n = WORKLOADS["cfg2"]["n"]
    return a


def encoder_cfg(args):
    cfg = inputs.CONFIGS[args.config]
    if args.pooling == "cls":
        cfg = inputs.EncoderConfig(**{**cfg.to_dict(), "pooling": inputs.POOL_CLS})
    return cfg


def workload(args, rank: int):
    """Batch workloads (cfg1-3): rank `rank`'s requests (lengths, generated, packed tokens)."""
    if args.total_requests > 0:
        # strong scaling: one request population for every N, rank r takes its contiguous slice
        full = argparse.Namespace(**{**vars(args), "n": args.total_requests, "total_requests": 0})
        L, gen, tokens = workload(full, 0)
        offs = inputs.offsets(L)
        a, b = rank * args.n, (rank + 1) * args.n
        return L[a:b].copy(), gen[a:b].copy(), tokens[offs[a]:offs[b]].copy()
    n = args.n
    seed = args.seed * 1000 + rank
    if args.lengths == "trace":
        L, gen, _ = inputs.trace_lengths(n, seed=seed)
    elif args.lengths == "uniform":
        L = inputs.uniform_lengths(n, seed=seed)
        gen = np.zeros(n, np.int32)
    elif args.lengths.startswith("fixed:"):
        L = np.full(n, int(args.lengths.split(":")[1]), np.int32)
        gen = np.zeros(n, np.int32)
    else:
        raise SystemExit(f"unknown --lengths {args.lengths}")
    tokens = inputs.make_tokens(L, seed=seed)
    return L.astype(np.int32), gen.astype(np.int32), tokens


def table_population(args):
    """cfg5: the in-flight population (identical on every rank): per-slot lengths of the prompt +
    partial response, tokens generated so far, packed tokens and their offsets."""
    F = args.inflight
    seed = args.seed * 1000
    if args.lengths == "uniform":
        Lt = inputs.uniform_lengths(F, seed=seed)
        gen_t = np.zeros(F, np.int32)
    else:
        Lt, gen_t, _ = inputs.trace_lengths(F, seed=seed)
    tok_t = inputs.make_tokens(Lt, seed=seed)
    return Lt.astype(np.int32), gen_t.astype(np.int32), tok_t, inputs.offsets(Lt)


def due_windows(F: int, due: int):
    """Global slots of each iteration's due set: consecutive windows of `due` slots, wrapping, so
    every slot is re-predicted once per ceil(F / due) iterations (no slot is left without a
    prediction)."""
    nwin = -(-F // due)
    return [((k * due + np.arange(due)) % F).astype(np.int32) for k in range(nwin)]


def cost_bounds(L: np.ndarray, world: int, cfg) -> np.ndarray:
    """Cost-balanced contiguous split of the due set, computed by the library."""
    from paper_2505_09142_b200 import binding
    return binding.cost_split(L, world, cfg)


L2_BYTES = 126 * 2 ** 20


def residual_fp16(args) -> bool:
    """The residual stream the run uses: --residual, else the library default (elis.h
    ELIS_RESID_AUTO: fp16 with fp16 operands -- the AUTO precision for head dim 64 -- and no CLS-only layer)."""
    if args.residual:
        return args.residual == "fp16"
    d64 = inputs.CONFIGS[args.config].head_dim == 64
    return d64 and args.precision in (None, "fp16") and not args.cls_last_layer


def working_set_bytes(args, T_local):
    """Bytes one step touches: encoder weights (2 B), the fp32 head, and the activations the
    layers stream (hidden / qkv / ctx / GELU rows, 2 B each; fp32 residual when not residual16)."""
    cfg = inputs.CONFIGS[args.config]
    H, F, nl = cfg.hidden, cfg.intermediate, cfg.num_layers
    enc = 2 * (cfg.vocab_size * H + nl * (4 * H * H + 2 * H * F))
    head = 4 * (H * 1024 + 6 * 1024 * 1024 + 1024)
    act = T_local * (2 * (H + 3 * H + H + F) + (0 if residual_fp16(args) else 4 * H))
    return enc + head + act


def l2_policy(args, T_local):
    """(flush?, description): steps whose working set is not well above the 126 MB L2 get an L2
    flush (a 256 MB device memset, outside the per-step events) before every timed step."""
    ws = working_set_bytes(args, T_local)
    if ws > 2 * L2_BYTES:
        return False, f"no flush: per-step working set ~{ws / 2 ** 20:.0f} MB exceeds 2x the 126 MB L2"
    return True, (f"L2 flushed before every timed step (256 MB memset outside the per-step events): working set "
                  f"~{ws / 2 ** 20:.0f} MB would otherwise stay L2-resident")


def config_desc(args, T_step, world):
    """The workload (identical in both arms: only the workload's own numbers).  T_step: tokens
    re-encoded per iteration over all GPUs (cfg5: averaged over the due windows)."""
    if args.inflight > 0:
        wl = (f"cfg5: {args.config} encoder, {args.inflight} requests in flight ({args.lengths} lengths); each "
              f"iteration re-predicts the {args.due} due requests (jobs returning from a 50-token window) into the "
              f"in-flight table and selects batch_cap {args.cap} over all {args.inflight} cached keys"
              + (f"; due set split over {world} GPUs at the quantiles of its encoder cost, predictions all-gathered "
                 f"to every GPU, the same select on each" if world > 1 else ""))
        d = {"workload": wl, "encoder": args.config, "inflight": args.inflight, "due_per_iteration": args.due,
             "tokens_per_iteration": int(T_step), "lengths": args.lengths, "batch_cap": args.cap}
    else:
        cfgno = {"tiny": 1, "base": 2, "large": 3}[args.config]
        wl = (f"cfg{cfgno}: {args.config} encoder re-predicting {args.n} in-flight requests per GPU "
              f"({args.lengths} lengths) + ISRTF select batch_cap {args.cap}"
              + (f" over {world}x{args.n}" if world > 1 else ""))
        d = {"workload": wl, "encoder": args.config, "inflight": args.n * world, "requests_per_gpu": args.n,
             "tokens_per_gpu_step": int(T_step // max(world, 1)), "lengths": args.lengths, "batch_cap": args.cap}
    d.update({
        "pooling": args.pooling + (" (last layer on CLS rows only)" if args.cls_last_layer else ""),
        "parallelism": f"request-sharded dp{world}" if world > 1 else "single GPU",
        "l2": l2_policy(args, T_step // max(world, 1))[1],
    })
    return d


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML every 10 ms (the
    timed region of the default run is ~0.2 s), else nvidia-smi every 200 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    NVML_BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.sm, self.mx, self.reasons = [], None, set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[gpu_index]) if vis and vis.split(",")[0].isdigit() else gpu_index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
        self.mx = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except AttributeError:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for k, b in self.NVML_BITS.items():
            if bits & b:
                self.reasons.add(k)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                              "-i", str(self.idx)], capture_output=True, text=True, timeout=5).stdout
        for line in out.strip().splitlines():
            r = [x.strip() for x in line.split(",")]
            self.sm.append(float(r[1]))
            self.mx = float(r[2])
            for k, v in zip(self.NAMES, r[5:9]):
                if v.lower().startswith("active"):
                    self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.01 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml 10 ms" if self._nvml else "nvidia-smi 200 ms"}


# ----------------------------------------------------------------------------- roofline
MUFU_EX2_PER_CLK_SM = 16   # MUFU ex2 lanes per SM per clock (B200_PROFILING.md; the softmax's exp bound)
FP32_LANES_SM = 128        # FP32 FMA lanes per SM
SMS = 148
SUSTAINED_AFTER_S = 4.0    # timed regions at least this long are compared with the sustained tensor peak


def step_work(cfg, T: float, n: float, sum_L2: float, table: int, residual16: bool, cls_last_layer: bool = False):
    """Algorithmic work of ONE step per kernel class: {name: (launches, tensor FLOP,
    HBM bytes, MUFU exps, FP32-ALU FLOP)} per launch.  T / n / sum_L2: tokens, requests and sum of
    L_i^2 of the step's predict call on this GPU; table: slots keyed and selected."""
    H, F, nl, nh = cfg.hidden, cfg.intermediate, cfg.num_layers, cfg.num_heads
    Tr = (T * (nl - 1) + n) / nl if cls_last_layer else T   # rows per out / FFN launch
    rs = 2 if residual16 else 4                              # residual-stream bytes per element
    hd = [H] + [cfg.head_hidden] * (cfg.head_layers - 2)
    return {
        "gemm_qkv": (nl, 2.0 * T * H * 3 * H, 0.0, 0.0, 0.0),
        "gemm_out": (nl, 2.0 * Tr * H * H, 0.0, 0.0, 0.0),
        "gemm_ffn1": (nl, 2.0 * Tr * H * F, 0.0, 0.0, 0.0),
        "gemm_ffn2": (nl, 2.0 * Tr * F * H, 0.0, 0.0, 0.0),
        # Q, K, V read and ctx written once (2 B each), S = QK^T and PV on the tensor pipe, one exp per score
        "attention": (nl, 4.0 * H * sum_L2, 8.0 * H * T, nh * sum_L2, 0.0),
        "embed_ln": (1, 0.0, T * (4 + 2 * H + 2 * H + (0 if residual16 else 4 * H)), 0.0, 0.0),
        "pool": (1, 0.0, T * H * rs + n * H * 4, 0.0, 0.0),
        "head_fc": (len(hd), 0.0, 0.0, 0.0, 2.0 * n * sum(k * cfg.head_hidden for k in hd) / len(hd)),
        "select_keys": (1, 0.0, table * (4 + 4 + 8), 0.0, 0.0),
        "select_topk": (1, 0.0, table * 8, 0.0, 0.0),
    }


def peaks_for(peaks: dict, timed_s: float, fp8: bool = False):
    """Roofline denominators from MEASURED_PEAKS.json: the burst tensor peak for a timed region
    shorter than SUSTAINED_AFTER_S (the bench's regions are sub-second), else the sustained one."""
    burst = peaks.get("bf16_tflops") or 1678.0
    sust = peaks.get("bf16_tflops_sustained") or burst
    kind = "burst" if timed_s < SUSTAINED_AFTER_S else "sustained"
    t = (burst if kind == "burst" else sust) * (2.0 if fp8 else 1.0)
    clk = (peaks.get("sm_max_mhz") or 1965.0) * 1e6
    return {
        "tensor_tflops": t, "tensor_kind": kind, "tensor_burst": burst, "tensor_sustained": sust,
        "hbm_gbs": peaks.get("hbm_gbs") or 6528.7,
        "mufu_gexp_s": MUFU_EX2_PER_CLK_SM * SMS * clk / 1e9,
        "fp32_tflops": FP32_LANES_SM * 2 * SMS * clk / 1e12,
        "source": "MEASURED_PEAKS.json (bf16 %s TF/s, HBM copy GB/s); MUFU %d ex2/clk/SM and FP32 %d lanes/SM x "
                  "148 SMs x sm_max_mhz (B200_PROFILING.md unit counts)" % (kind, MUFU_EX2_PER_CLK_SM, FP32_LANES_SM),
    }


def ideal_ms(work, pk):
    """Time at the roofline of one launch: the largest of its tensor / HBM / MUFU / FP32 bounds."""
    _, fl, by, ex, alu = work
    return 1e3 * max(fl / (pk["tensor_tflops"] * 1e12), by / (pk["hbm_gbs"] * 1e9), ex / (pk["mufu_gexp_s"] * 1e9),
                     alu / (pk["fp32_tflops"] * 1e12))


def roofline_report(prof: dict, steps: int, work: dict, pk: dict, ms_step: float, traffic: dict, traffic_key: str):
    """roofline object for the dominant kernel class + the whole-step fraction (sum of per-kernel ideal
    times at the measured peaks / measured step time) + attention's tensor / HBM / MUFU fractions."""
    name, (ms, cnt) = max(prof.items(), key=lambda kv: kv[1][0])
    avg_s = ms / cnt / 1e3
    w = work.get(name)
    if w is None:
        return {"kernel": name, "bound": "latency", "avg_launch_us": round(avg_s * 1e6, 2)}
    _, fl, by, ex, alu = w
    if fl > 0:
        bound, unit, achieved, peak = "tensor", "TFLOP/s", fl / avg_s / 1e12, pk["tensor_tflops"]
    elif alu > 0:
        bound, unit, achieved, peak = "alu", "TFLOP/s", alu / avg_s / 1e12, pk["fp32_tflops"]
    else:
        bound, unit, achieved, peak = "hbm", "GB/s", by / avg_s / 1e9, pk["hbm_gbs"]
    total_meas = sum(v[0] for v in prof.values()) / steps
    ideal = sum(ideal_ms(w2, pk) * w2[0] for k, w2 in work.items() if k in prof)
    out = {"kernel": name, "bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": unit,
           "frac": round(achieved / peak, 4), "traffic": traffic.get(f"{traffic_key}/{name}"),
           "traffic_key": f"{traffic_key}/{name}", "peak_source": pk["source"],
           "peak_kind": pk["tensor_kind"] if bound == "tensor" else "measured" if bound == "hbm" else "derived",
           "avg_launch_us": round(avg_s * 1e6, 2), "launches_per_step": round(cnt / steps, 2),
           "share_of_step": round(ms / steps / ms_step, 4) if ms_step else None,
           "algorithmic_per_launch": {"flop": fl, "bytes": by, "exp": ex, "fp32_flop": alu},
           "step_ideal_ms": round(ideal, 4), "step_frac": round(ideal / ms_step, 4) if ms_step else None,
           "step_frac_kernels_only": round(ideal / total_meas, 4) if total_meas else None}
    if bound == "tensor":
        out["frac_vs_sustained"] = round(achieved / (pk["tensor_sustained"] * (peak / pk["tensor_burst"]
                                                                                if pk["tensor_kind"] == "burst" else 1)), 4)
    if "attention" in prof and "attention" in work:
        a_ms, a_n = prof["attention"]
        a_s = a_ms / a_n / 1e3
        _, afl, aby, aex, _ = work["attention"]
        out["attention"] = {"avg_launch_us": round(a_s * 1e6, 2),
                            "tensor_frac": round(afl / a_s / 1e12 / pk["tensor_tflops"], 4),
                            "hbm_frac": round(aby / a_s / 1e9 / pk["hbm_gbs"], 4),
                            "mufu_frac": round(aex / a_s / 1e9 / pk["mufu_gexp_s"], 4),
                            "traffic": traffic.get(f"{traffic_key}/attention")}
    out["per_kernel_frac"] = {k: round(ideal_ms(work[k], pk) * work[k][0] / (v[0] / steps), 4)
                              for k, v in sorted(prof.items()) if k in work and v[0] > 0}
    return out


def load_json(path):
    try:
        with open(os.path.join(ROOT, path)) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------------------- oracle (CPU)
def cpu_sample_idx(L: np.ndarray, k: int):
    order = np.argsort(L, kind="stable")
    return sorted(set(order[np.linspace(0, len(L) - 1, k).astype(int)].tolist()))


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads") or 1) for i in threadpool_info()) or os.cpu_count()
    except Exception:
        return os.cpu_count()


def time_oracle_predict(cfg, W, L, tokens, idx):
    from oracle import head as ohead
    t0 = time.perf_counter()
    ohead.predict(tokens, L, W, cfg, requests=idx)
    return time.perf_counter() - t0, int(np.sum(L[idx]))


def time_oracle_select(pred, gen, cap):
    from oracle.select import isrtf_select
    t0 = time.perf_counter()
    isrtf_select(np.asarray(pred, np.float32), gen, cap)
    return time.perf_counter() - t0


def oracle_population(args):
    """The workload the oracle samples: (lengths, generated, tokens, per-step request count, select size)."""
    if args.inflight > 0:
        Lt, gen_t, tok_t, _ = table_population(args)
        return Lt, gen_t, tok_t, args.due, args.inflight
    L, gen, tokens = workload(args, 0)
    return L, gen, tokens, len(L), len(L)


def oracle_rate(cfg, W, args, per_step: int, steps: int, warmup: int):
    """Oracle predictions/s on length-stratified samples of the workload: each step predicts
    `per_step` requests and runs one oracle select over the whole key set (the table's cached keys
    are seeded stand-ins: inputs.random_predictions); the select's time is charged per due request
    (t_select x per_step / due), i.e. value = 1 / (oracle time per prediction + select time / due)."""
    L, gen, tokens, due, nsel = oracle_population(args)
    keys = inputs.random_predictions(nsel, seed=1, kind="spread") if args.inflight > 0 else None
    pool = cpu_sample_idx(L, max(per_step * (steps + warmup), per_step))
    t_pred, t_sel, reqs, toks = 0.0, 0.0, 0, 0
    for s in range(warmup + steps):
        idx = pool[(s * per_step) % len(pool):(s * per_step) % len(pool) + per_step] or pool[:per_step]
        dt, nt = time_oracle_predict(cfg, W, L, tokens, idx)
        if keys is not None:
            ds = time_oracle_select(keys, gen, args.cap)
        else:
            ds = time_oracle_select(np.zeros(len(idx), np.float32) + 1.0, gen[idx], args.cap)
        if s >= warmup:
            t_pred += dt
            t_sel += ds * (len(idx) / due if keys is not None else 1.0)
            reqs += len(idx)
            toks += nt
    total = t_pred + t_sel
    return reqs / total, total, reqs, toks


# ----------------------------------------------------------------------------- main arms
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if share_gpu():
        local = 0
    return world, rank, local


def share_gpu() -> bool:
    """ELIS_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 with a gloo control plane, so the
    N > 1 code path (peer-memory transport over CUDA IPC, barriers, max over ranks, the JSON line)
    can be exercised on a one-GPU box.  Its timings are meaningless (the ranks share one GPU)."""
    return os.environ.get("ELIS_BENCH_SHARE_GPU") == "1"


def _ctl(t):
    """Tensor for a control-plane collective: CUDA under NCCL, host memory under gloo."""
    return t.cpu() if share_gpu() else t


def step_tokens(args, world):
    """Tokens re-encoded per iteration over all GPUs (cfg5: the average over the due windows)."""
    if args.inflight > 0:
        Lt, _, _, _ = table_population(args)
        return int(round(np.mean([Lt[w].sum() for w in due_windows(args.inflight, args.due)])))
    return int(sum(workload(args, r)[0].sum() for r in range(world)))


def run_reference(args):
    """Reference arm = the fp64 oracle (this tier has no reference implementation), timed on the host
    cores on a bounded sample of the same workload per step (oracle_rate)."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    cfg = encoder_cfg(args)
    W = inputs.make_weights(cfg, seed=0)
    per_step = 2
    value, total, reqs, toks = oracle_rate(cfg, W, args, per_step, args.steps, args.warmup)
    sample = (f"{per_step} length-stratified requests of the workload per step, fp64 numpy oracle "
              + (f"+ one oracle select over all {args.inflight} keys per step, charged {per_step}/{args.due} of it "
                 f"(the step's work is {args.due} predictions + one select)" if args.inflight > 0 else
                 "+ oracle select over them") + f"; {toks} tokens total")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / args.steps, 3),
           "higher_is_better": True, "scaling": "strong" if args.inflight > 0 or args.total_requests else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_desc(args, step_tokens(args, max(world, args.gpus)), max(world, args.gpus)),
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "tokens_per_s": round(toks / total, 2)}
    print(json.dumps(out), flush=True)


class Shard:
    """One rank's per-step inputs: device tokens / lengths / slots of each due window (cfg5) or of
    the batch workload, plus pinned host copies for the end-to-end call."""

    def __init__(self, torch, tokens, lengths, slots=None):
        self.n = int(len(lengths))
        self.T = int(lengths.sum())
        self.L = lengths
        self.h_tok = torch.from_numpy(np.ascontiguousarray(tokens, np.int32)).pin_memory()
        self.h_len = torch.from_numpy(np.ascontiguousarray(lengths, np.int32)).pin_memory()
        self.d_tok = self.h_tok.cuda()
        self.d_len = self.h_len.cuda()
        self.h_slots = None if slots is None else torch.from_numpy(np.ascontiguousarray(slots, np.int32)).pin_memory()
        self.d_slots = None if slots is None else self.h_slots.cuda()


def run_elis(args):
    import torch
    import torch.distributed as dist

    from paper_2505_09142_b200 import binding

    world, rank, local = dist_env()
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    table_mode = args.inflight > 0
    if args.total_requests > 0 and not table_mode:  # strong scaling: fixed total work split over the ranks
        if args.total_requests % world:
            raise SystemExit(f"--total-requests {args.total_requests} is not a multiple of {world} GPUs")
        args.n = args.total_requests // world
    torch.cuda.set_device(local)
    if world > 1:
        if share_gpu():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = encoder_cfg(args)
    W = inputs.make_weights(cfg, seed=0)
    st = torch.cuda.current_stream()
    d_ids = torch.empty(args.cap, dtype=torch.int32, device="cuda")
    d_cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    kw = dict(device=local, cls_last_layer=args.cls_last_layer)
    if args.precision:
        kw["precision"] = args.precision
    if args.residual:
        kw["residual16"] = args.residual == "fp16"

    if table_mode:
        # In-flight table (the Priority Buffer keeps every slot's cached prediction; only the due set
        # is re-predicted each iteration).  Every rank holds the whole table and
        # the whole population; the due window is split at the quantiles of its encoder cost
        # (elis_cost_split) and rank r encodes its slice.
        F = args.inflight
        Lt, gen_t, tok_t, offs = table_population(args)
        wins = due_windows(F, args.due)
        shards, bounds_all = [], []
        for sl in wins:
            b = cost_bounds(Lt[sl], world, cfg)
            bounds_all.append(b)
            mine = sl[b[rank]:b[rank + 1]]
            toks = np.concatenate([tok_t[offs[i]:offs[i + 1]] for i in mine]) if len(mine) else np.zeros(0, np.int32)
            shards.append(Shard(torch, toks, Lt[mine], mine))
        max_T = max(max(sh.T for sh in shards), 1)
        max_n = args.due      # every rank uses the same max_requests (the exchange's pair capacity)
        P = binding.Predictor(cfg, inputs.flatten_weights(cfg, W), max_T, max_n, **kw)
        d_table = torch.zeros(F, device="cuda")
        d_gen = torch.from_numpy(gen_t).cuda()
        T_step_global = float(np.mean([Lt[sl].sum() for sl in wins]))
    else:
        L, gen, tokens = workload(args, rank)
        sh = Shard(torch, tokens, L)
        shards = [sh]
        P = binding.Predictor(cfg, inputs.flatten_weights(cfg, W), sh.T, sh.n, **kw)
        d_gen = torch.from_numpy(gen).cuda()
        d_pred = torch.empty(sh.n, device="cuda")
        T_step_global = None

    args.transport_used = "none"
    if world > 1:
        ok = 0
        if args.transport == "peer":
            # symmetric regions mapped through CUDA IPC; every rank must agree on the transport
            try:
                h = P.peer_export(rank, world)
                hs = [None] * world
                dist.all_gather_object(hs, h)
                P.peer_attach(hs)
                ok = 1
            except binding.ElisError as e:
                print(f"[rank {rank}] peer transport unavailable: {e}", file=sys.stderr)
        flag = _ctl(torch.tensor([ok], dtype=torch.int32, device="cuda"))
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            args.transport_used = "peer (NVLink stores + epoch flags in fused kernels)"
        else:
            uid = binding.nccl_unique_id() if rank == 0 else bytes(128)
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            P.dist_attach(rank, world, obj[0])   # the last attach wins: NCCL transport
            args.transport_used = "nccl all-gather"

    if table_mode:
        def step(s=None, wi=0):
            s = s or st
            sh = shards[wi]
            if world > 1:
                P.predict_remaining_dist(sh.d_tok, sh.d_len, sh.T, d_table, sh.d_slots, stream=s)
            else:
                P.predict_remaining(sh.d_tok, sh.d_len, sh.T, d_table, out_slot=sh.d_slots, stream=s)
            P.isrtf_select(d_table, d_gen, args.cap, d_ids, out_count=d_cnt, stream=s)
        # prefill: every window once fills every slot's cached prediction (also the warm-up)
        for wi in range(len(shards)):
            step(wi=wi)
        nwin = len(shards)
    else:
        def step(s=None, wi=0):
            s = s or st
            P.predict_remaining(sh.d_tok, sh.d_len, sh.T, d_pred, stream=s)
            if world > 1:
                P.isrtf_select_dist(d_pred, d_gen, rank * sh.n, args.cap, d_ids, out_count=d_cnt, stream=s)
            else:
                P.isrtf_select(d_pred, d_gen, args.cap, d_ids, out_count=d_cnt, stream=s)
        nwin = 1
    for k in range(max(args.warmup, 3)):
        step(wi=k % nwin)
    if P.sync_status() != 0:
        raise SystemExit("device error during warm-up: " + binding.lib().elis_last_error().decode())

    # ---------------- CUDA graphs of one step per due window (same library calls, side stream)
    graph, graph_note = None, "off"
    if args.graph == "on":
        try:
            cs = torch.cuda.Stream()
            cs.wait_stream(st)
            graphs = []
            for wi in range(nwin):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                    step(cs, wi)
                graphs.append(g)
            st.wait_stream(cs)
            for g in graphs[:2]:
                g.replay()
            torch.cuda.synchronize()
            if P.sync_status() != 0:
                raise RuntimeError(binding.lib().elis_last_error().decode())
            graph = graphs
            graph_note = (f"on (timed steps replay CUDA graphs of the step's launches: {len(graphs)} graph"
                          f"{'s, one per due window' if len(graphs) > 1 else ''})")
        except Exception as e:  # eager timing, say why
            graph, graph_note = None, f"off (capture failed: {str(e)[:120]})"
            torch.cuda.synchronize()

    def run_step(k):
        wi = k % nwin
        if graph is not None:
            graph[wi].replay()
        else:
            step(wi=wi)

    # ---------------- timed region (device events on the launching stream)
    T_local_avg = float(np.mean([shards[k % nwin].T for k in range(args.steps)]))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sampler = ClockSampler(local) if rank == 0 else None
    flush, _ = l2_policy(args, T_local_avg)
    flush_buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if flush else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.__enter__()
    t_wall0 = time.perf_counter()
    ev[0].record(st)
    for k in range(args.steps):
        if flush:
            flush_buf.zero_()
            ev[k].record(st)   # the step's own start: the flush is not timed
        run_step(k)
        ev_end[k].record(st)
        if not flush:
            ev[k + 1].record(st)
    torch.cuda.synchronize()
    timed_wall_s = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    if sampler:
        sampler.__exit__()
    # ---------------- per-kernel breakdown: the same K steps again, eager, with CUDA events around
    # every launch on the launching stream (the library profiler); kept out of the headline timing
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    P.profile_enable(True)
    evp = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    launches0 = P.launch_count()
    evp[0].record(st)
    for k in range(args.steps):
        step(wi=k % nwin)
    evp[1].record(st)
    torch.cuda.synchronize()
    launches = P.launch_count() - launches0   # the graphs replay exactly the eager steps' launches
    prof = P.profile_read()
    P.profile_enable(False)
    ms_step_profiled = evp[0].elapsed_time(evp[1]) / args.steps
    per_step = [ev[k].elapsed_time(ev_end[k]) for k in range(args.steps)]
    total_ms = sum(per_step) if flush else ev[0].elapsed_time(ev[-1])
    t = _ctl(torch.tensor([total_ms], dtype=torch.float64, device="cuda"))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_step = total_ms / args.steps
    units_per_step = args.due if table_mode else world * sh.n
    value = units_per_step * args.steps / (total_ms / 1e3)
    if T_step_global is None:
        Tg = _ctl(torch.tensor([float(sh.T)], dtype=torch.float64, device="cuda"))
        if world > 1:
            dist.all_reduce(Tg, op=dist.ReduceOp.SUM)
        T_step_global = float(Tg.item())

    # ---------------- end to end through the public C ABI with HOST buffers: every step copies its
    # due tokens / lengths / slots in and the selected ids out, synchronised per step
    h_ids = torch.empty(args.cap, dtype=torch.int32).pin_memory()
    h_cnt = torch.empty(1, dtype=torch.int32).pin_memory()
    if table_mode:
        def e2e_step(k):
            sh = shards[k % nwin]
            P.iteration_table_host(sh.h_tok, sh.h_len, sh.h_slots, d_table, d_gen, args.cap, h_ids, h_cnt, stream=st)
        h2d = float(np.mean([4 * (shards[k % nwin].T + 2 * shards[k % nwin].n) for k in range(args.steps)]))
    else:
        h_gen = torch.from_numpy(gen).pin_memory()
        goff = rank * sh.n if world > 1 else -1

        def e2e_step(k):
            P.iteration_host(sh.h_tok, sh.h_len, h_gen, args.cap, h_ids, h_cnt, global_offset=goff, stream=st)
        h2d = float(4 * sh.T + 8 * sh.n)
    for k in range(2):
        e2e_step(k)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        e2e_step(k)
    e2e_s = _ctl(torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda"))
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = units_per_step * args.steps / float(e2e_s.item())
    if P.sync_status() != 0:
        raise SystemExit("device error: " + binding.lib().elis_last_error().decode())

    out = None
    if rank == 0:
        prec = P.c.precision
        prec_name = {v: k for k, v in binding.PRECISION.items()}.get(prec, "auto")
        if prec_name == "auto":
            prec_name = "fp16" if cfg.head_dim == 64 else "bf16"
        r16 = residual_fp16(args)
        pk = peaks_for(load_json("MEASURED_PEAKS.json"), total_ms / 1e3, fp8=prec_name == "fp8")
        prof_steps = {k: v for k, v in prof.items()}
        n_avg = float(np.mean([shards[k % nwin].n for k in range(args.steps)]))
        sL2 = float(np.mean([float(np.sum(shards[k % nwin].L.astype(np.float64) ** 2)) for k in range(args.steps)]))
        work = step_work(cfg, T_local_avg, n_avg, sL2, args.inflight if table_mode else sh.n, r16, args.cls_last_layer)
        tkey = f"{args.workload}{'' if world == 1 else f'-n{world}'}/{prec_name}{'-r16' if r16 else ''}"
        roof = roofline_report(prof_steps, args.steps, work, pk, ms_step, load_json("profiles/traffic.json"), tkey)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "ms_per_step_p10_p50_p90": [round(float(np.percentile(per_step, q)), 4) for q in (10, 50, 90)],
            "higher_is_better": True,
            "scaling": "strong" if table_mode or args.total_requests > 0 else "weak",
            "vs_baseline": None,
            "dtype": {"bf16": "bf16", "fp16": "fp16",
                      "fp8": "fp8_e4m3 GEMMs (bf16 attention, fp32 residual/LN/head)"}[prec_name],
            "data": "synthetic (seeded trace-shaped lengths, uniform token ids, random-init BGE weights)",
            "config": config_desc(args, T_step_global, world),
            "precision": {"operands": prec_name, "residual_stream": "fp16" if r16 else "fp32",
                          "head": "fp32", "select_keys": "fp32"},
            "timing": {"cuda_graph": graph_note, "timed_region_s": round(total_ms / 1e3, 4),
                       "timed_region_wall_s": round(timed_wall_s, 4),
                       "transport": args.transport_used if world > 1 else None},
            "sharding": ({"due_split": "elis_cost_split quantiles of c(L)", "rank0_requests_avg": round(n_avg, 1),
                          "rank0_tokens_avg": round(T_local_avg, 1),
                          "rank_requests_window0": np.diff(bounds_all[0]).tolist()} if table_mode and world > 1
                         else None),
            "tokens_per_s": round(T_step_global * args.steps / (total_ms / 1e3), 1),
            "roofline": roof,
            "kernels_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in sorted(prof.items())},
            "kernels_pass_ms_per_step": round(ms_step_profiled, 4),
            "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(4 * args.cap + 4),
                    "call": "elis_iteration_table_host" if table_mode else "elis_iteration_host"},
            "gpu_launches": int(launches),
            "clocks": sampler.summary() if sampler else None,
        }
        if not args.no_cpu_baseline and world == 1:
            v, tot, reqs, toks = oracle_rate(cfg, W, args, args.cpu_sample, 1, 0)
            out["cpu_baseline"] = {
                "value": round(v, 4), "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
                "sample": f"{reqs} length-stratified requests of this workload ({toks} tokens) encoded by the fp64 "
                          f"numpy oracle" + (f" + one oracle select over all {args.inflight} keys charged "
                                             f"{reqs}/{args.due} of it" if table_mode else " + oracle select"),
                "seconds": round(tot, 2)}
    P.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.cls_last_layer and args.pooling != "cls":
        raise SystemExit("--cls-last-layer needs --pooling cls")
    if args.residual == "fp16" and (args.precision not in (None, "fp16") or args.cls_last_layer):
        raise SystemExit("--residual fp16 needs fp16 operands and no --cls-last-layer")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_elis(args)


if __name__ == "__main__":
    main()
