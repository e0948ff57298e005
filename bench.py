#!/usr/bin/env python
"""Benchmark of the DELTA decode-step attention stack (BASELINE.json metric).

One "step" = one decode step through the whole attention stack (all layers: fused append
+ decode for every layer, score + top-k after each Delta layer), i.e. all §8(a) rows, on a
synthetic cache shaped like the configured model.  Default workload: BASELINE configs[1]
(DeepSeek-R1-Distill-Llama-8B shape, batch 1, context 32K, token budget 2K, page-level
selection, Delta = {2, 16, 25}).  The context grows by one token per step exactly as in
decoding: the first timed step has s = 32768 tokens after its append.

value      = attended-KV GB/s of the DELTA stack over the whole job: algorithmic KV bytes
             read by all ranks' steps / max-over-ranks device time.
e2e        = same metric through delta_decode_step_host (pinned host inputs copied H2D
             and outputs D2H inside the timed region).
roofline   = the dominant kernel (full-cache decode of one layer) timed live with CUDA
             events, algorithmic bytes / average launch time, against MEASURED_PEAKS.json.
Also reported: DELTA and Full stack µs per step, their speedup, and the byte ratio.

Multi-GPU (torchrun): each rank owns whole sequences (batch sharding) — no collective on
the data path; barrier + max-over-ranks timing only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-step attention µs and attended-KV HBM GB/s @32K ctx; DELTA vs full speedup"

CONFIGS = {
    # name: model shape, per-config batch, context, budget, schedule (R14), scaling mode
    "c1": dict(workload="DeepSeek-R1-Distill-Llama-8B shape (32L, 32q/8kv, d128, bf16) b=1 ctx 32K budget 2K",
               L=32, m=32, g=8, d=128, batch=1, ctx=32768, k=2048, delta=[2, 16, 25], F=2, scaling="weak"),
    "c2": dict(workload="DeepSeek-R1-Distill-Qwen-7B shape (28L, 28q/4kv, d128, bf16) b=32 ctx 16K budget 4K",
               L=28, m=28, g=4, d=128, batch=32, ctx=16384, k=4096, delta=[2, 14, 22], F=2, scaling="strong"),
    "c3": dict(workload="Llama-8B shape b=1 ctx 128K budget 2K, KV sequence-sharded over the GPUs (NCCL LSE "
                        "partial merge + global top-k candidate merge)",
               L=32, m=32, g=8, d=128, batch=1, ctx=131072, k=2048, delta=[2, 16, 25], F=2, scaling="strong",
               shard="seq"),
    "c4": dict(workload="Qwen3-14B shape (40L, 40q/8kv, d128, bf16) ctx 32K budget 2K, 8 sequences per GPU "
                        "(the 8xB200 config's per-GPU share of batch 64; 43 GB of KV per GPU)",
               L=40, m=40, g=8, d=128, batch=8, ctx=32768, k=2048, delta=[2, 6, 35], F=2, scaling="weak"),
}
S_SINK, L_WIN, PAGE = 4, 32, 16


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ clocks sampling
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons through NVML every ~2 ms while the
    timed region runs (nvidia-smi's 100 ms floor is longer than a short timed region)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.sm, self.bits = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None
        self.err = None

    def _run(self, hd):
        import pynvml
        try:
            while True:
                self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM)))
                self.bits |= int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd))
                self._first.set()
                if self._stop.wait(0.002):
                    break
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            self._first.set()

    def start(self):
        """NVML is initialised here, before the timed region; returns once the sampler has taken
        its first sample, so the samples cover the region that follows."""
        self._first = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            hd = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(hd, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            return
        self.t = threading.Thread(target=self._run, args=(hd,), daemon=True)
        self.t.start()
        self._first.wait(timeout=2.0)
        self.sm.clear()  # keep only samples taken from here on
        self.bits = 0

    def stop(self):
        self._stop.set()
        if self.t is not None:
            self.t.join(timeout=5)
        if self.err and not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"], "samples": 0}
        reasons = sorted(n for bit, n in self.REASONS.items() if self.bits & bit and n != "gpu_idle")
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm), "source": "NVML, 2 ms period, during the timed region"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy, measured on this pool)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# ------------------------------------------------------------------ byte model
def step_bytes(c, s: int, batch: int, sparse_tokens: int) -> dict:
    """Algorithmic bytes of one step per the byte model: FULL/SELECT layers read all s tokens'
    K+V; SPARSE layers read |tokens(rho)| rows + plan indices; append writes one row."""
    row = c["g"] * c["d"] * 2 * 2                       # K+V bytes per token per layer (bf16)
    n_full = c["F"] + len(c["delta"])
    n_sparse = c["L"] - n_full
    n_units = sparse_tokens // PAGE
    full = n_full * s * row
    sparse = n_sparse * (sparse_tokens * row + n_units * 4)
    append = c["L"] * row
    return {"delta": batch * (full + sparse + append), "full_stack": batch * c["L"] * (s * row) + batch * append}


def sparse_token_count(s: int, k: int) -> int:
    """|tokens(rho)| in page mode: sink page(s) + window pages + k/P pages (R1, R6)."""
    n_pages = -(-s // PAGE)
    forced = set(range(0, (S_SINK - 1) // PAGE + 1)) | set(range(max(0, s - L_WIN) // PAGE, n_pages))
    sel_pages = min(n_pages, len(forced) + k // PAGE)
    toks = sel_pages * PAGE
    if (n_pages - 1) in forced and s % PAGE:
        toks -= PAGE - s % PAGE   # the partial last page holds only s % P tokens
    return toks


# ------------------------------------------------------------------ reference arm (oracle)
def run_reference(args, c):
    """The oracle (fp64 C, OpenMP) timed on host cores, on a bounded sample per step."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import synth
    cores = os.cpu_count() or 1
    s = c["ctx"]
    scale = float(np.float32(1.0 / math.sqrt(c["d"])))
    seed = 2511
    sample_layers = [0, c["delta"][0], c["delta"][0] + 1]   # one FULL, one Delta, one SPARSE layer
    # inputs (generation is not timed)
    kvs, qs = {}, {}
    for l in sample_layers:
        K = synth.kv_rows(seed, l, 0, 0, s, c["g"], c["d"], "bf16", "k")
        V = synth.kv_rows(seed, l, 0, 0, s, c["g"], c["d"], "bf16", "v")
        kvs[l] = oracle.SeqKV.from_contiguous(K, V, PAGE)
        qs[l] = synth.q_rows(seed, l, 0, s, c["m"], c["d"], "bf16")
    cfg = oracle.StackConfig(num_layers=c["L"], m=c["m"], g=c["g"], d=c["d"], page_size=PAGE,
                             num_full_prefix=c["F"], select_layers=c["delta"], budget_k=c["k"], n_sink=S_SINK,
                             n_window=L_WIN, select_block=PAGE, scale=scale)
    row = c["g"] * c["d"] * 2 * 2

    def one_step():
        t0 = time.perf_counter()
        byts = 0
        oracle.decode_heads(qs[sample_layers[0]], kvs[sample_layers[0]], s, scale, nthreads=cores)
        byts += s * row
        _, _, alpha = oracle.decode_heads(qs[sample_layers[1]], kvs[sample_layers[1]], s, scale, want_alpha=True,
                                          nthreads=cores)
        _, units = oracle.select_from_alpha(cfg, alpha, s)
        byts += s * row
        toks = oracle.units_to_tokens(units, PAGE, s)
        oracle.decode_heads(qs[sample_layers[2]], kvs[sample_layers[2]], toks, scale, nthreads=cores)
        byts += toks.size * row
        return time.perf_counter() - t0, byts

    for _ in range(args.warmup):
        one_step()
    tot_t, tot_b = 0.0, 0
    for _ in range(args.steps):
        dt, b = one_step()
        tot_t += dt
        tot_b += b
    value = tot_b / tot_t / 1e9
    sample = (f"per step: layers {sample_layers} (FULL, Delta incl. score+top-k, SPARSE) of one sequence at "
              f"s={s}; fp64 oracle, {cores} OpenMP threads; KV generation untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot_t / args.steps, 3),
        "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator)", "config": {"workload": c["workload"], "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(c, cores=None):
    """Oracle timed on this host's cores on a bounded sample (one FULL layer of one sequence
    at the config's context): attended-KV GB/s of the oracle."""
    import numpy as np
    import oracle
    import synth
    cores = cores or os.cpu_count() or 1
    s = c["ctx"]
    scale = float(np.float32(1.0 / math.sqrt(c["d"])))
    K = synth.kv_rows(2511, 0, 0, 0, s, c["g"], c["d"], "bf16", "k")
    V = synth.kv_rows(2511, 0, 0, 0, s, c["g"], c["d"], "bf16", "v")
    kv = oracle.SeqKV.from_contiguous(K, V, PAGE)
    q = synth.q_rows(2511, 0, 0, s, c["m"], c["d"], "bf16")
    reps, t = 0, 0.0
    while t < 10.0:  # about 10 s of CPU work
        t0 = time.perf_counter()
        oracle.decode_heads(q, kv, s, scale, nthreads=cores)
        t += time.perf_counter() - t0
        reps += 1
    byts = reps * s * c["g"] * c["d"] * 4
    # the same layer on one thread (the core count and a 1-thread number)
    t1, reps1 = 0.0, 0
    while t1 < 2.0:
        t0 = time.perf_counter()
        oracle.decode_heads(q, kv, s, scale, nthreads=1)
        t1 += time.perf_counter() - t0
        reps1 += 1
    # the other roles of a step, sampled on the same sequence, for an extrapolated oracle step
    # time at this config (C2-C4 are too large to run whole on the host)
    cfg_o = oracle.StackConfig(num_layers=c["L"], m=c["m"], g=c["g"], d=c["d"], page_size=PAGE,
                               num_full_prefix=c["F"], select_layers=c["delta"], budget_k=c["k"], n_sink=S_SINK,
                               n_window=L_WIN, select_block=PAGE, scale=scale)
    t_delta, reps_d, toks = 0.0, 0, None
    while t_delta < 3.0 or reps_d < 2:
        t0 = time.perf_counter()
        _, _, alpha = oracle.decode_heads(q, kv, s, scale, want_alpha=True, nthreads=cores)
        _, units = oracle.select_from_alpha(cfg_o, alpha, s)
        t_delta += time.perf_counter() - t0
        reps_d += 1
        toks = oracle.units_to_tokens(units, PAGE, s)
    t_sp, reps_s = 0.0, 0
    while t_sp < 1.0 or reps_s < 3:
        t0 = time.perf_counter()
        oracle.decode_heads(q, kv, toks, scale, nthreads=cores)
        t_sp += time.perf_counter() - t0
        reps_s += 1
    t_f1, t_d1, t_s1 = t / reps, t_delta / reps_d, t_sp / reps_s
    n_sp = c["L"] - c["F"] - len(c["delta"])
    per_seq = c["F"] * t_f1 + len(c["delta"]) * t_d1 + n_sp * t_s1
    cpu_model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu_model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": round(byts / t / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
            "sample": f"{reps} x one FULL layer (all {c['m']} heads) of one sequence at s={s}, fp64, "
                      f"{t:.1f} s of CPU time; KV generation untimed",
            "value_1thread": round(reps1 * s * c["g"] * c["d"] * 4 / t1 / 1e9, 4), "cpu": cpu_model,
            "oracle_step_s_extrapolated": {
                "delta": round(c["batch"] * per_seq, 3), "full": round(c["batch"] * c["L"] * t_f1, 3),
                "per_sequence_layer_s": {"full": round(t_f1, 4), "delta_incl_score_topk": round(t_d1, 4),
                                         "sparse": round(t_s1, 5)},
                "how": (f"extrapolated: batch {c['batch']} x (F={c['F']} full + {len(c['delta'])} Delta (full + score + "
                        f"top-k) + {n_sp} sparse layers), each timed on one sampled sequence/layer at s={s}")}}


# ------------------------------------------------------------------ our arm
def run_ours(args, c):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2510_09883_b200 as d200
    import synth
    from synth import device as sd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    seq_shard = c.get("shard") == "seq" and world > 1
    if c["scaling"] == "weak" or seq_shard:
        batch = c["batch"]
    else:
        batch = max(1, c["batch"] // world)
    nccl_ids = [None, None]
    if seq_shard:  # rank 0 creates one NCCL id per handle (DELTA stack, Full stack); all ranks join
        obj = [[d200.nccl_unique_id(), d200.nccl_unique_id()] if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_ids = obj[0]
    W, K = args.warmup, args.steps
    s_first = c["ctx"]                        # s after the append of the first timed step
    s_pre = s_first - W - 1                   # tokens in the cache before warm-up
    max_seq = s_first + K + PAGE
    seed = 2511 if seq_shard else 2511 + 1000 * rank  # batch sharding: every rank its own sequences

    def make_cfg(full: bool, quest: bool = False, raas: bool = False, budget: int | None = None):
        return d200.DeltaConfig(num_layers=c["L"], num_q_heads=c["m"], num_kv_heads=c["g"], head_dim=c["d"],
                                max_batch=batch, max_seq_len=max_seq,
                                num_full_prefix=c["L"] if full else c["F"],
                                select_layers=[] if (full or quest or raas) else c["delta"],
                                budget_k=budget or c["k"], n_sink=S_SINK, n_window=L_WIN, select_block=PAGE,
                                shard_world=world if seq_shard else 1, shard_rank=rank if seq_shard else 0,
                                nccl_id=nccl_ids[1 if full else 0],
                                policy=(d200.POLICY_QUEST if quest else d200.POLICY_RAAS if raas else d200.POLICY_DELTA))

    cfg = make_cfg(False)
    bt = torch.from_numpy(synth.block_table(seed, batch, cfg.max_pages))
    delta = d200.DeltaStack.allocate(cfg, bt, device=dev)
    # the Full stack shares the pools and block table (same library, every layer FULL)
    fcfg = make_cfg(True)
    _, fws = d200.query_sizes(fcfg)
    full = d200.DeltaStack(fcfg, delta.kv_pool, delta.block_table,
                           torch.zeros(fws, dtype=torch.uint8, device=dev))
    # the paper's comparison policy Quest (NEXT-1) on the same pools: every layer >= F selects
    # its own pages from min/max key representatives (its own workspace)
    quest = None
    if not seq_shard:
        qcfg = make_cfg(False, quest=True)
        _, qws = d200.query_sizes(qcfg)
        quest = d200.DeltaStack(qcfg, delta.kv_pool, delta.block_table,
                                torch.zeros(qws, dtype=torch.uint8, device=dev))
    # the paper's eviction baseline RaaS (NEXT-4) on the same pools (its own retained sets)
    raas = None
    if not seq_shard:
        rcfg = make_cfg(False, raas=True)
        _, rws = d200.query_sizes(rcfg)
        raas = d200.DeltaStack(rcfg, delta.kv_pool, delta.block_table,
                               torch.zeros(rws, dtype=torch.uint8, device=dev))
    t0 = time.time()
    sd.fill_pools(delta.kv_pool, delta.block_table, seed, s_pre, batch, range(c["L"]))
    if quest is not None:
        quest.set_seq_lens([s_pre] * batch)
        quest.quest_build_reps(-1, batch)
    torch.cuda.synchronize()
    log(f"[rank {rank}] filled {delta.kv_pool.numel() * 2 / 2**30:.1f} GiB KV in {time.time() - t0:.1f}s "
        f"(batch {batch}, s_pre {s_pre})")

    L_, m, g, d = c["L"], c["m"], c["g"], c["d"]
    n_steps = W + K
    q_all = torch.empty((n_steps, L_, batch, m, d), dtype=torch.bfloat16, device=dev)
    k_all = torch.empty((n_steps, L_, batch, g, d), dtype=torch.bfloat16, device=dev)
    v_all = torch.empty_like(k_all)
    for i in range(n_steps):
        s = s_pre + 1 + i
        sd.fill_queries(q_all[i], seed, range(L_), [s] * batch)
        sd.fill_new_kv(k_all[i], v_all[i], seed, range(L_), [s - 1] * batch)
    out = torch.empty((L_, batch, m, d), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    stack_pct = {}

    # One set of device input buffers for every warm-up and timed step (q_all[W] etc. are fixed
    # views), so delta_decode_step captures its graph once, during warm-up, and the timed loop is
    # pure graph replays (asserted with the library's capture counter).  Each step still appends
    # its row at the next position (s grows by one per step).
    q_fix, k_fix, v_fix = q_all[W], k_all[W], v_all[W]

    def time_stack(stack, clocks=None):
        stack.set_seq_lens([s_pre] * batch)
        if stack is raas:
            stack.raas_reset(-1, batch, stream=stream)  # every page retained; warm-up steps evict to the budget
        with torch.cuda.stream(stream):
            for i in range(W):
                stack.decode_step(q_fix, k_fix, v_fix, out, stream=stream)
        stream.synchronize()
        launched0 = stack.kernels_launched
        captures0 = stack.graph_captures
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(K - 1)]  # per-step boundaries
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for j in range(K):
                stack.decode_step(q_fix, k_fix, v_fix, out, stream=stream)
                if j < K - 1:
                    evs[j].record(stream)
            ev1.record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        barrier()
        clk = clocks.stop() if clocks else None
        ms = ev0.elapsed_time(ev1)
        marks = [ev0] + evs + [ev1]
        steps_us = sorted(1e3 * marks[j].elapsed_time(marks[j + 1]) for j in range(K))
        pct = {"p50": round(steps_us[len(steps_us) // 2], 2), "p90": round(steps_us[min(K - 1, (9 * K) // 10)], 2)}
        stack_pct[id(stack)] = pct
        assert stack.graph_captures == captures0, "the timed region re-captured a graph (not pure replay)"
        return ms, stack.kernels_launched - launched0, clk

    clocks = ClockSampler(local)
    ms_delta, launches, clk = time_stack(delta, clocks)
    ms_full, _, _ = time_stack(full)
    ms_quest = time_stack(quest)[0] if quest is not None else None
    ms_raas = time_stack(raas)[0] if raas is not None else None
    for other in (quest, raas):
        if other is not None:
            e_other = other.get_error()
            assert e_other == 0, f"device error flag {e_other} (comparison stack)"
    err = delta.get_error()
    assert err == 0, f"device error flag {err}"

    # ---- budget sweep (PAPER.md:217-223's budget axis): DELTA(k) vs the same Full
    sweep = []
    for kb in ([int(x) for x in args.budget.split(",")] if args.budget else []):
        bcfg = make_cfg(False, budget=kb)
        _, bws = d200.query_sizes(bcfg)
        bst = d200.DeltaStack(bcfg, delta.kv_pool, delta.block_table, torch.zeros(bws, dtype=torch.uint8, device=dev))
        ms_b = time_stack(bst)[0]
        assert bst.get_error() == 0
        bst.close()
        bb = bf = 0
        for i in range(K):
            sb = step_bytes(c, s_first + i, batch, sparse_token_count(s_first + i, kb))
            bb += sb["delta"]
            bf += sb["full_stack"]
        sweep.append({"budget_k": kb, "delta_us": round(1e3 * ms_b / K, 2), "speedup_vs_full": round(ms_full / ms_b, 3),
                      "byte_ratio": round(bf / bb, 3), "speedup_target": round(0.8 * bf / bb, 3)})

    # max over ranks
    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_delta = max_over_ranks(ms_delta)
    ms_full = max_over_ranks(ms_full)
    if ms_quest is not None:
        ms_quest = max_over_ranks(ms_quest)
    if ms_raas is not None:
        ms_raas = max_over_ranks(ms_raas)

    # algorithmic bytes over the timed steps (s grows by one per step)
    byts_delta = byts_full = 0
    for i in range(K):
        s = s_first + i
        sb = step_bytes(c, s, batch, sparse_token_count(s, c["k"]))
        byts_delta += sb["delta"]
        byts_full += sb["full_stack"]
    tot_delta = byts_delta * (1 if seq_shard else world)  # sequence sharding: one sequence in total
    value = tot_delta / (ms_delta * 1e-3) / 1e9

    # ---- e2e through delta_decode_step_host (pinned host buffers, copies inside the region)
    qh = q_all[W:].cpu().pin_memory()
    kh = k_all[W:].cpu().pin_memory()
    vh = v_all[W:].cpu().pin_memory()
    oh = torch.empty((L_, batch, m, d), dtype=torch.float32).pin_memory()
    delta.set_seq_lens([s_first - 1] * batch)
    with torch.cuda.stream(stream):  # warm the host-step graphs (two staging slots) at the same context
        delta.decode_step_host(qh[0], kh[0], vh[0], oh, stream=stream)
        delta.decode_step_host(qh[1], kh[1], vh[1], oh, stream=stream)
    stream.synchronize()
    delta.set_seq_lens([s_first - 1] * batch)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(K):
            delta.decode_step_host(qh[i], kh[i], vh[i], oh, stream=stream)
        ev1.record(stream)
    stream.synchronize()
    barrier()
    ms_e2e = max_over_ranks(ev0.elapsed_time(ev1))
    e2e_value = tot_delta / (ms_e2e * 1e-3) / 1e9
    h2d = (qh[0].numel() + kh[0].numel() + vh[0].numel()) * 2
    d2h = oh.numel() * 4

    # ---- per-kernel timings, eager launches on `stream` (CUDA events on that stream).  The
    # state after the last e2e step is a consistent decode step at s_last, so every role may
    # be re-run without an append: FULL (layer 0), SELECT decode + delta_select (first Delta
    # layer), SPARSE (the layer after it, reusing that Delta layer's plan).
    s_last = s_first + K - 1
    reps = 50

    def time_calls(fn):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(stream):
            for _ in range(5):
                fn()
            ev[0].record(stream)
            for _ in range(reps):
                fn()
            ev[1].record(stream)
        stream.synchronize()
        return ev[0].elapsed_time(ev[1]) * 1e3 / reps

    dl = c["delta"][0]
    sp = dl + 1
    qW = q_all[W + K - 1]
    us_full = time_calls(lambda: delta.decode_layer(0, qW[0], out[0], stream=stream))
    us_sel_dec = time_calls(lambda: delta.decode_layer(dl, qW[dl], out[dl], stream=stream))
    us_select = time_calls(lambda: delta.select(dl, batch, stream=stream))
    us_sparse = time_calls(lambda: delta.decode_layer(sp, qW[sp], out[sp], stream=stream))
    err = delta.get_error()
    assert err == 0, f"device error flag {err} after per-kernel timing"
    kbytes = batch * s_last * g * d * 2 * 2
    n_sp_tok = sparse_token_count(s_last, c["k"])
    sp_bytes = batch * (n_sp_tok * g * d * 2 * 2 + (n_sp_tok // PAGE) * 4)
    peak, peak_src = measured_peaks()

    # ---- in-graph launch durations (the DELTA step is a graph of PDL-chained kernels; eager
    # back-to-back launches are not the same thing).  FULL: the Full stack's timed region is
    # nothing but FULL-layer launches -> region time / launches.  SPARSE: two graph-replayed
    # stacks on the same pools that differ only in their number of sparse layers (layer 0 SELECT
    # governing layers 1..n-1, with n = L and n = 4): (t_L - t_4) / (L - 4) sparse launches.
    def chain_us(n_layers):
        ccfg = d200.DeltaConfig(num_layers=n_layers, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=batch,
                                max_seq_len=max_seq, num_full_prefix=0, select_layers=[0], budget_k=c["k"],
                                n_sink=S_SINK, n_window=L_WIN, select_block=PAGE)
        _, cws = d200.query_sizes(ccfg)
        st_ = d200.DeltaStack(ccfg, delta.kv_pool, delta.block_table,  # layers [0, n) of the same pools
                              torch.zeros(cws, dtype=torch.uint8, device=dev))
        st_.set_seq_lens([s_pre] * batch)
        qn, kn, vn = q_fix[:n_layers], k_fix[:n_layers], v_fix[:n_layers]
        with torch.cuda.stream(stream):
            for _ in range(W):
                st_.decode_step(qn, kn, vn, out[:n_layers], stream=stream)
        stream.synchronize()
        cap0 = st_.graph_captures
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(K):
                st_.decode_step(qn, kn, vn, out[:n_layers], stream=stream)
            e1.record(stream)
        stream.synchronize()
        assert st_.graph_captures == cap0 and st_.get_error() == 0
        st_.close()
        return 1e3 * e0.elapsed_time(e1) / K

    us_full_graph = 1e3 * ms_full / (c["L"] * K) if not seq_shard else us_full
    us_sparse_graph = None
    if not seq_shard:
        us_sparse_graph = (chain_us(c["L"]) - chain_us(4)) / (c["L"] - 4.0)
    us_step = 1e3 * ms_delta / K
    n_fullcache = c["F"] + len(c["delta"])
    n_sparse_l = c["L"] - n_fullcache
    breakdown = {"full_cache_layers_us": round(n_fullcache * us_full_graph, 1)}
    if us_sparse_graph is not None:
        breakdown["sparse_layers_us"] = round(n_sparse_l * us_sparse_graph, 1)
        breakdown["select_and_rest_us"] = round(us_step - n_fullcache * us_full_graph - n_sparse_l * us_sparse_graph, 1)
        breakdown["select_per_delta_layer_us"] = round(breakdown["select_and_rest_us"] / len(c["delta"]), 2)
    breakdown["how"] = ("in-graph per-launch durations x launches: FULL from the Full stack's region, SPARSE from "
                        "(t(n=L) - t(n=4)) / (L - 4) of two graph-replayed SELECT+SPARSE chains on the same pools; "
                        "select_and_rest = the DELTA step minus both (the three score+top-k launches, and the "
                        "first sparse layer after each of them, which cannot prefetch its plan's pages)")

    # ---- pure-read roofline reference measured in this run (K10): stream the KV pool once
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    probe_bytes = delta.kv_pool.numel() * delta.kv_pool.element_size()
    probe_us = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            d200.read_bandwidth_probe(delta.kv_pool, sink, stream=stream)
            e1.record(stream)
        stream.synchronize()
        probe_us.append(1e3 * e0.elapsed_time(e1))
    pure_read_gbs = probe_bytes / (min(probe_us[1:]) * 1e-6) / 1e9
    NOMINAL_GBS = 8000.0  # north star "~8 TB/s"

    def roof(kernel, nbytes, us, how, share):
        a = nbytes / (us * 1e-6) / 1e9
        return {"bound": "hbm", "achieved": round(a, 1), "peak": peak, "unit": "GB/s", "frac": round(a / peak, 4),
                "frac_of_8tbs": round(a / NOMINAL_GBS, 4), "frac_of_pure_read": round(a / pure_read_gbs, 4),
                "kernel": kernel, "algorithmic_bytes_per_launch": int(nbytes), "avg_launch_us": round(us, 3),
                "share_of_step": round(share, 3) if share is not None else None, "measured": how,
                "peak_source": peak_src}

    roof_full = roof(f"FULL/SELECT layer: {delta.kernel_name(0, batch)}", kbytes,
                     us_full_graph, (f"in-graph: the Full stack's timed region, {c['L'] * K} FULL launches, device "
                                     f"time / launches; eager back-to-back {us_full:.3f} us"),
                     n_fullcache * us_full_graph / us_step)
    if us_sparse_graph is not None:
        roof_sparse = roof(f"SPARSE layer: {delta.kernel_name(sp, batch)}", sp_bytes, us_sparse_graph,
                           f"in-graph: (t(n={c['L']}) - t(n=4)) / {c['L'] - 4} of two SELECT+SPARSE chains; eager {us_sparse:.3f} us",
                           n_sparse_l * us_sparse_graph / us_step)
    else:
        roof_sparse = roof("SPARSE layer kernel, one layer (eager)", sp_bytes, us_sparse, "eager back-to-back", None)
    # DRAM traffic per launch from one ncu --set full capture of the same kernels at C1
    # (profiles/r2/ncu_traffic.json); other configs: not captured (null)
    roof_full["traffic"] = roof_sparse["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "r2", "ncu_traffic.json")
    if os.path.exists(prof) and args.config == "c1":
        try:
            tr = json.load(open(prof))
            roof_full["traffic"] = tr.get("full", {}).get("dram_bytes_per_launch")
            roof_sparse["traffic"] = tr.get("sparse", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
    # "roofline" = the kernel with the largest share of the DELTA step's time
    dominant = roof_full if (roof_sparse["share_of_step"] or 0) <= roof_full["share_of_step"] else roof_sparse
    kernels = {
        "full_layer_us": round(us_full, 3), "full_layer_gbs": round(kbytes / (us_full * 1e-6) / 1e9, 1),
        "select_layer_decode_us": round(us_sel_dec, 3), "select_topk_us": round(us_select, 3),
        "sparse_layer_us": round(us_sparse, 3), "sparse_layer_gbs": round(sp_bytes / (us_sparse * 1e-6) / 1e9, 1),
        "sparse_layer_bytes": sp_bytes, "note": "eager launches back to back (PDL), %d reps, s=%d" % (reps, s_last),
    }
    if rank == 0:
        log(f"DELTA {1e3 * ms_delta / K:.1f} us/step, Full {1e3 * ms_full / K:.1f} us/step, "
            f"speedup {ms_full / ms_delta:.3f}x; Quest {1e3 * ms_quest / K if ms_quest else 0:.1f} us/step; "
            f"RaaS {1e3 * ms_raas / K if ms_raas else 0:.1f} us/step; "
            f"kernels {kernels}")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    byte_ratio = byts_full / byts_delta
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": round(ms_delta / K, 5),
        "higher_is_better": True,
        "scaling": c["scaling"],
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded counter-based N(0,1) K/V/Q, bf16; scattered block table)",
        "config": {"workload": c["workload"], "per_rank_batch": batch, "global_batch": batch * world,
                   "context": f"s = {s_first}..{s_first + K - 1} tokens after append (grows 1/step)",
                   "budget_k": c["k"], "n_sink": S_SINK, "n_window": L_WIN, "select_block": PAGE,
                   "delta_layers": c["delta"], "full_prefix": c["F"], "parallelism": (f"sequence-shard x{world} (NCCL)" if seq_shard else f"batch-shard x{world}"),
                   "l2": "inputs larger than L2: >= 861 MB of KV read per step vs 126 MB L2 (no flush)"},
        "decode_step_us": round(1e3 * ms_delta / K, 2),
        "decode_step_us_pct": stack_pct.get(id(delta)),
        "full_stack_us_pct": stack_pct.get(id(full)),
        "full_stack_us": round(1e3 * ms_full / K, 2),
        "speedup_vs_full": round(ms_full / ms_delta, 3),
        "quest_stack_us": round(1e3 * ms_quest / K, 2) if ms_quest else None,
        "quest_speedup_vs_full": round(ms_full / ms_quest, 3) if ms_quest else None,
        "raas_stack_us": round(1e3 * ms_raas / K, 2) if ms_raas else None,
        "byte_ratio": round(byte_ratio, 3),
        "speedup_target": round(0.8 * byte_ratio, 3),
        "full_stack_gbs": round(byts_full * (1 if seq_shard else world) / (ms_full * 1e-3) / 1e9, 2),
        "roofline": dominant,
        "roofline_full": roof_full,
        "roofline_sparse": roof_sparse,
        "pure_read_gbs": round(pure_read_gbs, 1),
        "step_breakdown": breakdown,
        "kernels": kernels,
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(ms_e2e / K, 5)},
        "budget_sweep": sweep or None,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(c)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--budget", default="", help="comma-separated token budgets for a DELTA(k) sweep, e.g. "
                                                 "1024,2048,4096,8192 (reported as budget_sweep)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    c = CONFIGS[args.config]
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference(args, c)
        return
    run_ours(args, c)


if __name__ == "__main__":
    main()
