#!/usr/bin/env python
"""OSCAR hot-path benchmark on B200 (see DESIGN.md §8 for every definition used here).

Workload (N=1, BASELINE.json configs[1], "C2"): Llama-3-8B-shaped GQA decode — 32 q / 8 kv
heads, d=128, 2-bit codes, G=64, batch 16, 32k context, 32 layers.  One timed STEP = one
decode step through all 32 layers: quantize_append of the 16 new K/V rows (overwriting slot
L-1 so the context stays 32768) + attend(q) over the packed paged cache, per layer.  Each
layer's pool is 335.5 MB (> 126 MB L2) and the 32 pools are visited in turn, so no input is
L2-resident between uses.  The pools are filled beforehand by our own prefill
quantize_append (timed: the append half of the metric), with rotations produced by our own
on-device calibration (timed: C3 per-rank shard).

value = algorithmic bytes of all ranks' timed steps / max-over-ranks device time (GB/s).
Multi-GPU (torchrun, NCCL): every rank runs the same per-GPU workload (weak scaling); the
calibration covariances are all-reduced over NCCL (the path's only exchange step).
`--impl reference`: the CPU oracle timed on bounded samples of the same workload (rank 0).
"""
import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packed-KV decode attention HBM GB/s (% of 8 TB/s); quantize-append tokens/s"
NOMINAL_HBM_GBS = 8000.0
B_, L_, HQ, HKV, D, BITS, G, P = 16, 32768, 32, 8, 128, 2, 64, 64
TOKHEAD_BYTES = 2 * (D * BITS // 8 + 4 * (D // G))                    # = 80 for b=2, G=64
APPEND_BYTES_PER_TOKHEAD = 2 * D * 2 + TOKHEAD_BYTES + 8 // HKV       # 593 B


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops_sustained", 1417.2)), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback"


def bf16_burst_peak():
    """Dense bf16 TFLOP/s of a kernel timed alone: MEASURED_PEAKS.json's burst figure."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured (burst)"
    except Exception:
        return 2250.0, "nominal (no MEASURED_PEAKS.json)"


# ------------------------------------------------------------------ clocks sampler (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
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
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in self.REASONS.items():
                    if bits & k and k != 0x1:
                        self.reasons.add(v)
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
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def ncu_kernel(name):
    """(duration µs, DRAM bytes) of one kernel from the committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            j = json.load(f)
        for k, v in j["kernels"].items():
            if k.startswith(name):
                d = v[0]
                scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
                return d["duration"] * scale.get(d.get("duration_unit", "us"), 1.0), d["traffic_bytes"]
    except Exception:
        pass
    return None


def ncu_traffic(kernels):
    """DRAM bytes per launch (read + write) of the named kernels, summed, from the committed
    `ncu --set full` capture (profiles/ncu_traffic.json, written by tools/ncu_traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            j = json.load(f)
        tot = 0.0
        for k in kernels:
            runs = [v for name, v in j["kernels"].items() if name.startswith(k)]
            if not runs:
                return None
            tot += max(x["traffic_bytes"] for x in runs[0])
        return tot
    except Exception:
        return None


def oracle_timed(fn):
    """Run an oracle call on ONE host thread (BLAS pinned to 1 thread: the oracle's per-token
    loops are single-threaded anyway, so the core count reported is the one used)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        t0 = time.perf_counter()
        r = fn()
        return r, time.perf_counter() - t0


def cpu_threads():
    return 1


# The JSON line goes to the process's original stdout; everything else written to fd 1 (library
# banners such as NCCL's version line) is sent to stderr, so stdout carries exactly one line.
_JSON_OUT = None


def claim_stdout():
    global _JSON_OUT
    if _JSON_OUT is None:
        sys.stdout.flush()
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(obj) + "\n")
    out.flush()


# ------------------------------------------------------------------ reference (CPU oracle) arm
def run_reference(args, rank):
    if rank != 0:
        return
    import numpy as np
    import oracle as O
    from paper_2605_17757_b200 import synth
    rng = np.random.default_rng(1)
    fmt = O.PageFormat(D, BITS, G, P)
    max_pages = L_ // P
    # one (sequence, kv-head) unit per step: 32768 tokens of one KV head, its 4 query heads
    pool = synth.random_pool(rng, max_pages, 1, fmt.page_bytes, fmt.meta_off, P * (D // G))
    RK, RV = synth.gen_rotation(rng, 1, D), synth.gen_rotation(rng, 1, D)
    q = synth.gen_decode_q(rng, 1, HQ // HKV, D)
    pt = np.arange(max_pages, dtype=np.int32)[None]
    unit_bytes = L_ * TOKHEAD_BYTES + 2 * (HQ // HKV) * D * 2
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        for _ in range(args.warmup):
            O.attend(q, pt, [L_], pool, RK, RV, fmt, 1)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            O.attend(q, pt, [L_], pool, RK, RV, fmt, 1)
        dt = time.perf_counter() - t0
    gbs = unit_bytes * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle",
                         "sample": "per step: 1 sequence x 1 kv head (4 q heads) x 32768 tokens "
                                   "of the C2 decode workload (1/128 of one layer-step)"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def workload_config(args):
    return {"workload": "C2: Llama-3-8B-shaped GQA decode on 1 B200 per rank (BASELINE.json configs[1])",
            "batch": B_, "context": L_, "q_heads": HQ, "kv_heads": HKV, "head_dim": D, "bits": BITS,
            "group": G, "page": P, "layers": args.layers, "parallelism": f"weak x{args.gpus} (per-rank C2)",
            "l2": "inputs larger than L2: 335.5 MB pool per layer, layers visited in turn"}


# ------------------------------------------------------------------ C4 leg
C4_B, C4_L, C4_HQ, C4_HKV, C4_LAYERS = 16, 131072, 64, 8, 4


def c4_leg(args, world, rank, dev, gen, RK_all, RV_all, hbm_peak, peak_kind):
    """Decode attention at C4 (H_q 64 / H_kv 8, g = 8, 2-bit, G = 64, B = 16, L = 131072): each rank
    owns 8/N KV heads and their query heads for all sequences (no collective on the path)."""
    import torch
    from paper_2605_17757_b200 import binding as Bnd
    from paper_2605_17757_b200 import synth
    from paper_2605_17757_b200.parallel import barrier, kv_head_shard, max_over_ranks
    kv_lo, kv_hi, q_lo, q_hi = kv_head_shard(C4_HKV, C4_HQ, rank, world) if C4_HKV % world == 0 else \
        (0, max(1, C4_HKV // world), 0, max(1, C4_HKV // world) * (C4_HQ // C4_HKV))
    hkv, hq = kv_hi - kv_lo, q_hi - q_lo
    o = Bnd.Oscar(Bnd.Config(num_q_heads=hq, num_kv_heads=hkv, bits=BITS, group_size=G, page_size=P))
    o.set_variant(args.variant)
    max_pages = C4_L // P
    pools = [torch.empty((C4_B * max_pages, hkv, o.page_bytes()), dtype=torch.uint8, device=dev)
             for _ in range(C4_LAYERS)]
    pt = torch.arange(C4_B * max_pages, dtype=torch.int32, device=dev)
    pt = pt[torch.randperm(C4_B * max_pages, generator=gen, device=dev)].reshape(C4_B, max_pages).contiguous()
    # this rank's KV heads [kv_lo, kv_hi) and their rotations (parallel.kv_head_shard)
    RK = [RK_all[l % RK_all.shape[0], kv_lo:kv_hi].contiguous() for l in range(C4_LAYERS)]
    RV = [RV_all[l % RV_all.shape[0], kv_lo:kv_hi].contiguous() for l in range(C4_LAYERS)]
    chunk = 4 * 8192                       # prefill in 32k-token slabs (bounded staging memory)
    for l in range(C4_LAYERS):
        for c0 in range(0, C4_B * C4_L, chunk):
            tok = torch.arange(c0, c0 + chunk, device=dev)
            b, pos = tok // C4_L, tok % C4_L
            slots = (pt[b, pos // P].long() * P + pos % P).contiguous()
            o.quantize_append(synth.torch_keys(gen, chunk, hkv, D, dev), synth.torch_values(gen, chunk, hkv, D, dev),
                              slots, RK[l], RV[l], pools[l])
    qs = [synth.torch_decode_q(gen, C4_B, hq, D, dev) for _ in range(C4_LAYERS)]
    seq = torch.full((C4_B,), C4_L, dtype=torch.int32, device=dev)
    ws = torch.empty(o.attend_workspace_bytes(C4_B, max_pages), dtype=torch.uint8, device=dev)
    out = torch.empty((C4_B, hq, D), dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        for l in range(C4_LAYERS):
            o.attend(qs[l], pt, seq, pools[l], RK[l], RV[l], ws, out)
    torch.cuda.synchronize(); barrier(world)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(5, args.steps)
    a.record()
    for _ in range(reps):
        for l in range(C4_LAYERS):
            o.attend(qs[l], pt, seq, pools[l], RK[l], RV[l], ws, out)
    b_.record(); torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b_), world) / (reps * C4_LAYERS)
    rank_bytes = C4_B * C4_L * hkv * TOKHEAD_BYTES + 2 * C4_B * hq * D * 2
    cpu = None
    if rank == 0 and world == 1 and not getattr(args, "no_cpu", False):
        # oracle: 1 sequence x 1 KV head (its 8 query heads) x 131072 tokens of layer 0
        import numpy as np
        import oracle as O
        fmt = O.PageFormat(D, BITS, G, P)
        sub = pools[0][pt[0].long(), :1].cpu().numpy()
        qn = qs[0][0:1, :C4_HQ // C4_HKV].float().cpu().numpy()
        (ref, _), dt = oracle_timed(lambda: O.attend(qn, np.arange(max_pages, dtype=np.int32)[None], [C4_L], sub,
                                                     RK[0][:1].cpu().numpy(), RV[0][:1].cpu().numpy(), fmt, 1))
        unit_bytes = C4_L * TOKHEAD_BYTES + 2 * (C4_HQ // C4_HKV) * D * 2
        cpu = {"value": unit_bytes / dt / 1e9, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": "layer 0, sequence 0, kv head 0 (8 q heads) x 131072 tokens (1/128 of a layer-step)",
               "seconds": dt}
    del pools
    r = {"config": f"C4: B={C4_B}, L={C4_L}, H_q/H_kv = {C4_HQ}/{C4_HKV} (g=8), b={BITS}, G={G}; "
                   f"kv heads [{kv_lo}, {kv_hi}) on rank {rank} of {world} (parallel.kv_head_shard); "
                   f"{C4_LAYERS} layer pools in turn",
         "attend_us": ms * 1e3, "GBps_per_rank": rank_bytes / ms / 1e6,
         "GBps_aggregate": rank_bytes * world / ms / 1e6,
         "roofline": {"bound": "hbm", "achieved": rank_bytes / ms / 1e6, "peak": hbm_peak, "unit": "GB/s",
                      "frac": rank_bytes / ms / 1e6 / hbm_peak,
                      "traffic": ncu_traffic(["attend_prologue_kernel<8>", "attend_partial_mma<2, 8, 2, 1>",
                                              "attend_merge_kernel<8>"]),
                      "traffic_source": "profiles/ncu_traffic.json (ncu --set full of the C4 launch, per launch)",
                      "kernel": "oscar_attend (prologue+partial+merge), g = 8",
                      "algorithmic_bytes_per_launch": rank_bytes, "peak_kind": peak_kind}}
    if cpu:
        r["cpu_baseline"] = cpu
    return r


def c5_leg(args, dev, hbm_peak, subset=False):
    """b in {2,3,4} x G in {32,64,128} x B in {1,16,64,256} decode at L = 32768
    (Llama-3-8B shape, random packed pools of the page FORMAT), and prefill-append of 4096 tokens
    per sequence for B in {1, 16, 64}.  Median of 7 calls after 2 warm-up calls.  subset=True (the
    default bench run): G = 64, B in {1, 16}, every b — the full sweep is `--c5-only`."""
    import torch
    from paper_2605_17757_b200 import binding as Bnd
    from paper_2605_17757_b200 import synth
    gen = torch.Generator(device=dev).manual_seed(4)
    L, pts = 32768, []

    def med(fn, reps=7):
        for _ in range(2):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record(); fn(); b.record()
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]

    RK, RV = synth.torch_rotation(gen, HKV, D, dev), synth.torch_rotation(gen, HKV, D, dev)
    for bits in (2, 3, 4):
        for g in ((64,) if subset else (32, 64, 128)):
            o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=bits, group_size=g, page_size=P))
            o.set_variant(args.variant)
            tok_b = 2 * (D * bits // 8 + 4 * (D // g))
            for B in ((1, 16) if subset else (1, 16, 64, 256)):
                mp = L // P
                pool = synth.torch_random_pool(gen, B * mp, HKV, o.page_bytes(), 2 * P * (D * bits // 8),
                                               P * (D // g), dev)
                pt = torch.randperm(B * mp, generator=gen, device=dev).to(torch.int32).reshape(B, mp).contiguous()
                seq = torch.full((B,), L, dtype=torch.int32, device=dev)
                q = synth.torch_decode_q(gen, B, HQ, D, dev)
                ws = torch.empty(o.attend_workspace_bytes(B, mp), dtype=torch.uint8, device=dev)
                out = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=dev)
                ms = med(lambda: o.attend(q, pt, seq, pool, RK, RV, ws, out))
                byt = B * L * HKV * tok_b + 2 * B * HQ * D * 2
                pts.append({"leg": "decode", "bits": bits, "G": g, "B": B, "L": L, "us": ms * 1e3,
                            "GBps": byt / ms / 1e6, "frac": byt / ms / 1e6 / hbm_peak})
                del pool
                if B <= 64:
                    T = B * 4096
                    K, V = synth.torch_keys(gen, T, HKV, D, dev), synth.torch_values(gen, T, HKV, D, dev)
                    npg = B * 4096 // P
                    pool = torch.empty((npg, HKV, o.page_bytes()), dtype=torch.uint8, device=dev)
                    slots = torch.randperm(npg, generator=gen, device=dev).repeat_interleave(P) * P + \
                        torch.arange(P, device=dev).repeat(npg)
                    ms = med(lambda: o.quantize_append(K, V, slots, RK, RV, pool))
                    byt = T * HKV * (2 * D * 2 + tok_b + 8 // HKV)
                    pts.append({"leg": "prefill_append", "bits": bits, "G": g, "B": B, "tokens": T,
                                "us": ms * 1e3, "tokens_per_s": T / ms * 1e3, "GBps": byt / ms / 1e6,
                                "frac": byt / ms / 1e6 / hbm_peak})
                    del pool, K, V
            torch.cuda.synchronize()
    return {"config": "C5 sweep (SURVEY §8(d)): Llama-3-8B shape (32 q / 8 kv heads, d 128), page 64; decode "
                      "attend at L = 32768 over random packed pools; prefill-append 4096 tokens per sequence "
                      "into randomly placed pages" + ("; subset G = 64, B in {1, 16} (full: --c5-only)"
                                                      if subset else ""), "peak_GBps": hbm_peak, "points": pts}


def c1_leg(args, dev):
    """SURVEY §8(d) C1 end to end (the correctness config, oracle in seconds): one KV head,
    d = 128, 4-bit codes, G = 32, P = 64.  calibrate on the 256 tokens' queries with causal
    S·V computed on the device (NEXT-3) -> quantize_append of the 256 K/V rows -> attend for 64
    queries whose page tables all point at the 4 pages (the page indirection).  The oracle runs
    the same steps on the host with the GPU's rotations (R is not comparable elementwise,
    reading Z12) and its own S·V; reported: GPU and oracle times and the fp32-output max-abs."""
    import numpy as np
    import torch
    import oracle as O
    from paper_2605_17757_b200 import binding as Bnd
    from paper_2605_17757_b200 import synth
    rng = np.random.default_rng(7)
    N, B1 = 256, 64
    Qn = synth.gen_queries(rng, N, 1, 1, D)
    Kn = synth.gen_keys(rng, N, 1, D)
    Vn = synth.gen_values(rng, N, 1, D)
    qn = synth.gen_decode_q(rng, B1, 1, D)
    o = Bnd.Oscar(Bnd.Config(num_q_heads=1, num_kv_heads=1, bits=4, group_size=32, page_size=P))
    o.set_variant(args.variant)
    fmt = O.PageFormat(D, 4, 32, P)
    bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.bfloat16)
    Q, K, V, q = bf(Qn), bf(Kn), bf(Vn), bf(qn)
    pt = torch.arange(4, dtype=torch.int32, device=dev).repeat(B1, 1).contiguous()
    seq = torch.full((B1,), N, dtype=torch.int32, device=dev)
    slots = torch.arange(N, dtype=torch.int64, device=dev)
    SV = torch.empty((N, 1, D), dtype=torch.bfloat16, device=dev)
    acc = torch.zeros((1, 2, D, D), dtype=torch.float64, device=dev)
    RK = torch.empty((1, D, D), dtype=torch.float32, device=dev)
    RV = torch.empty_like(RK)
    pool = torch.zeros((4, 1, o.page_bytes()), dtype=torch.uint8, device=dev)
    ws = torch.empty(o.attend_workspace_bytes(B1, 4), dtype=torch.uint8, device=dev)
    out = torch.empty((B1, 1, D), dtype=torch.float32, device=dev)
    starts = torch.zeros(1, dtype=torch.int32, device=dev)

    def gpu_path():
        acc.zero_()
        o.calib_sv(Q, K, V, starts, SV)
        o.calib_accumulate(Q, SV, acc)
        o.calib_finalize(acc, 1, N, RK, RV)
        o.quantize_append(K, V, slots, RK, RV, pool)
        o.attend(q, pt, seq, pool, RK, RV, ws, out)

    for _ in range(3):
        gpu_path()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    gpu_path()
    b.record()
    torch.cuda.synchronize()
    rk, rv = RK.cpu().numpy(), RV.cpu().numpy()

    def oracle_path():
        sv = O.score_value(Qn, Kn, Vn, [N])
        accq, accs = O.cov_accumulate(Qn, 1), O.cov_accumulate(sv, 1)
        O.calibrate_from_sums(accq, accs, N)
        opool = np.zeros((4, 1, fmt.page_bytes), np.uint8)
        O.quantize_append(Kn, Vn, np.arange(N), rk, rv, fmt, opool)
        return O.attend(qn, np.tile(np.arange(4, dtype=np.int32), (B1, 1)), [N] * B1, opool, rk, rv, fmt, 1)[0]

    ref, dt = oracle_timed(oracle_path)
    return {"config": "C1: 1 kv head, d 128, 4-bit, G 32, P 64; calibrate(256 tokens, causal S·V on device) -> "
                      "quantize_append(256) -> attend(64 queries over the same 4 pages)",
            "gpu_ms": a.elapsed_time(b), "oracle_s": dt, "oracle_cores": cpu_threads(),
            "parity_max_abs_fp32_out": float(np.abs(out.cpu().numpy() - ref).max()), "parity_tolerance": 2e-3}


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="oscar", choices=["oscar", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--variant", type=int, default=0, help="0 = fastest kernels, 1 = simple reference kernels")
    ap.add_argument("--no-extras", action="store_true", help="skip calibration / prefill / e2e / cpu legs (ncu runs)")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (Llama-3-70B-shaped, 128k) decode leg")
    ap.add_argument("--c4-only", action="store_true", help="run only the C4 decode leg and print its dict")
    ap.add_argument("--c5-only", action="store_true", help="run only the C5 sweep (bits x G x B) and print it")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle (cpu_baseline) legs")
    ap.add_argument("--no-graph", action="store_true", help="time the step as plain stream launches only")
    args = ap.parse_args()
    claim_stdout()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank)

    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL's INFO log (nranks, transports, NVLS) goes to stderr with the rest of the library
        # output (claim_stdout), so a scaling run can be checked against it
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        dist.init_process_group("nccl", device_id=dev)
    elif not args.no_extras:
        # a 1-rank NCCL group, so the calibration all-reduce (the path's one collective) runs NCCL
        # at N = 1 too (a no-op sum, but the real code path)
        try:
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                    device_id=dev)
        except Exception as e:   # NCCL unavailable: the all-reduce is skipped at N = 1
            print(f"bench: 1-rank NCCL group not available ({e})", file=sys.stderr)
    from paper_2605_17757_b200 import binding as Bnd
    from paper_2605_17757_b200 import synth
    from paper_2605_17757_b200.parallel import allreduce_covariances, barrier, max_over_ranks

    hbm_peak, _, peak_kind = measured_peaks()
    if args.c5_only:
        if rank == 0:
            emit(c5_leg(args, dev, hbm_peak))
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    if args.c4_only:
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        RK = torch.stack([synth.torch_rotation(gen, HKV, D, dev) for _ in range(C4_LAYERS)])
        RV = torch.stack([synth.torch_rotation(gen, HKV, D, dev) for _ in range(C4_LAYERS)])
        r = c4_leg(args, world, rank, dev, gen, RK, RV, hbm_peak, peak_kind)
        if rank == 0:
            emit(r)
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    o = Bnd.Oscar(Bnd.Config(num_q_heads=HQ, num_kv_heads=HKV, bits=BITS, group_size=G, page_size=P))
    o.set_variant(args.variant)
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    NL = args.layers
    max_pages = L_ // P
    extras = {}
    launches_per_layer = 3    # decode_step: prologue (q rotation + append), partial, merge

    # ---------------- calibration: C3 per-rank shard (65536 tokens/layer, NL layers)
    calib_tokens = 65536
    RK_all = torch.empty((NL, HKV, D, D), dtype=torch.float32, device=dev)
    RV_all = torch.empty_like(RK_all)
    if not args.no_extras:
        Q = synth.torch_queries(gen, calib_tokens, HQ, HKV, D, dev)
        SV = synth.torch_sv(gen, calib_tokens, HQ, D, dev)
        acc = torch.zeros((NL, HKV, 2, D, D), dtype=torch.float64, device=dev)
        for l in range(2):  # warm
            o.calib_accumulate(Q, SV, acc[0])
        acc.zero_()
        torch.cuda.synchronize(); barrier(world)
        e0, e1, e2, e3 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e0.record()
        for l in range(NL):
            o.calib_accumulate(Q, SV, acc[l])
        e1.record()
        allreduce_covariances(acc, world)
        e2.record()
        info = torch.empty((NL * HKV, 2), dtype=torch.int32, device=dev)
        o.calib_finalize(acc, NL * HKV, calib_tokens * world * (HQ // HKV), RK_all, RV_all, None, info)
        e3.record()
        torch.cuda.synchronize()
        t_acc, t_ar, t_fin = e0.elapsed_time(e1), e1.elapsed_time(e2), e2.elapsed_time(e3)
        # on-device S·V for C_S (NEXT-3), one layer: 8 calibration sequences of 8192 tokens
        Kc = synth.torch_keys(gen, calib_tokens, HKV, D, dev)
        Vc = synth.torch_values(gen, calib_tokens, HKV, D, dev)
        starts = torch.arange(0, calib_tokens, 8192, dtype=torch.int32, device=dev)
        SVd = torch.empty_like(SV)
        o.calib_sv(Q, Kc, Vc, starts, SVd)
        es0, es1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es0.record()
        o.calib_sv(Q, Kc, Vc, starts, SVd)
        es1.record()
        # CalibrateClip (reading Z34) on 8192 rows of that layer, Table 10's 5-point grid
        RKc, RVc = RK_all[0].contiguous(), RV_all[0].contiguous()
        ec0, ec1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        o.calib_clip(Kc[:8192], Vc[:8192], RKc, RVc, acc[0], [0.88, 0.92, 0.96, 0.98, 1.0])
        ec0.record()
        _, rho_k, rho_v = o.calib_clip(Kc[:8192], Vc[:8192], RKc, RVc, acc[0], [0.88, 0.92, 0.96, 0.98, 1.0])
        ec1.record()
        torch.cuda.synchronize()
        t_sv, t_clip = es0.elapsed_time(es1), ec0.elapsed_time(ec1)
        sv_flops = 2 * 2 * HQ * D * (calib_tokens // 8192) * (8192 * 8193 // 2)
        del Kc, Vc, SVd
        sweeps = info.cpu().numpy()
        cpu_cal = None
        if rank == 0 and world == 1 and not args.no_cpu:
            import oracle as O
            ns = 16384                           # 1/4 of a layer's shard; extrapolated per token
            Qh = Q[:ns].float().cpu().numpy()
            SVh = SV[:ns].float().cpu().numpy()
            _, t_cov = oracle_timed(lambda: (O.cov_accumulate(Qh, HKV), O.cov_accumulate(SVh, HKV)))
            acc_h = acc[0].cpu().numpy()
            _, t_eig = oracle_timed(lambda: O.calibrate_from_sums(acc_h[:, 0], acc_h[:, 1], calib_tokens * (HQ // HKV)))
            t_all = t_cov * (calib_tokens / ns) * NL + t_eig * (NL * HKV * 2) / 16
            cpu_cal = {"value": 2 * ns * HQ * D * 2 / t_cov / 1e9, "unit": "GB/s", "cores": cpu_threads(),
                       "kind": "oracle", "sample": f"cov_accumulate of {ns} tokens x {HQ} q heads (Q and SV) of one "
                                                   f"layer + 16 eigensolves (8 kv heads x K,V), extrapolated",
                       "cov_seconds": t_cov, "eig_seconds_16": t_eig,
                       "extrapolated_seconds_per_rank_shard": t_all}
        cov_bytes = NL * 2 * calib_tokens * HQ * D * 2
        cov_flops = NL * 2 * calib_tokens * HQ * 2 * D * D
        extras["calibration"] = {
            "config": f"C3 shard: {calib_tokens} tokens/rank/layer x {NL} layers x {HKV} kv heads, "
                      f"{world} rank(s), then {NL * HKV * 2} 128x128 eigensolves",
            "accumulate_ms": t_acc, "accumulate_GBps": cov_bytes / t_acc / 1e6,
            "accumulate_TFLOPs": cov_flops / t_acc / 1e9,
            "allreduce_ms": t_ar, "allreduce_bytes": acc.numel() * 8,
            "allreduce_backend": (dist.get_backend() if dist.is_initialized() else "none (1 rank)"),
            "finalize_ms": t_fin, "jacobi_sweeps_max": int(sweeps.max()),
            "sv_ms_per_layer": t_sv, "sv_TFLOPs": sv_flops / t_sv / 1e9,
            "sv_config": f"causal S·V, {calib_tokens // 8192} sequences x 8192 tokens, {HQ} q-heads",
            "sv_roofline": {"bound": "tensor", "achieved": sv_flops / t_sv / 1e9, "peak": bf16_burst_peak()[0],
                            "unit": "TFLOP/s", "frac": sv_flops / t_sv / 1e9 / bf16_burst_peak()[0],
                            "traffic": ncu_traffic(["calib_sv_tc_kernel"]),
                            "kernel": "calib_sv_tc_kernel (tcgen05 + TMA), one layer",
                            "algorithmic_flops_per_launch": sv_flops, "peak_kind": bf16_burst_peak()[1]},
            "clip_ms_per_layer": t_clip, "clip_config": "8192 rows x 8 kv heads x K,V x 5 ratios",
            "clip_choice_layer0": [rho_k, rho_v],
            "roofline": {"bound": "hbm", "achieved": cov_bytes / t_acc / 1e6, "peak": hbm_peak, "unit": "GB/s",
                         "frac": cov_bytes / t_acc / 1e6 / hbm_peak,
                         "traffic": ncu_traffic(["cov_accum_tc_kernel"]),
                         "kernel": "cov_accum_tc_kernel (tcgen05 + TMA), per layer launch",
                         "algorithmic_bytes_per_launch": cov_bytes // NL, "peak_kind": peak_kind},
        }
        if cpu_cal:
            extras["calibration"]["cpu_baseline"] = cpu_cal
        del Q, SV, acc
    else:
        for l in range(NL):
            RK_all[l] = synth.torch_rotation(gen, HKV, D, dev)
            RV_all[l] = synth.torch_rotation(gen, HKV, D, dev)

    # ---------------- prefill: fill NL layer pools with our quantize_append (timed on layer 0)
    page_bytes = o.page_bytes()
    pools = [torch.empty((B_ * max_pages, HKV, page_bytes), dtype=torch.uint8, device=dev) for _ in range(NL)]
    page_table = torch.arange(B_ * max_pages, dtype=torch.int32, device=dev).reshape(B_, max_pages)
    page_table = page_table.reshape(-1)[torch.randperm(B_ * max_pages, generator=gen, device=dev)].reshape(B_, max_pages).contiguous()
    pos = torch.arange(L_, device=dev)
    pre_slots = (page_table[:, pos // P].long() * P + (pos % P)).reshape(-1).contiguous()   # [B*L]
    Tpre = B_ * L_
    Kp = synth.torch_keys(gen, Tpre, HKV, D, dev)
    Vp = synth.torch_values(gen, Tpre, HKV, D, dev)
    for l in range(NL):
        o.quantize_append(Kp, Vp, pre_slots, RK_all[l], RV_all[l], pools[l])
    torch.cuda.synchronize()
    if not args.no_extras:
        reps = 5
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        ea.record()
        for r in range(reps):
            o.quantize_append(Kp, Vp, pre_slots, RK_all[r % NL], RV_all[r % NL], pools[r % NL])
        eb.record(); torch.cuda.synchronize()
        t = ea.elapsed_time(eb) / reps
        t = max_over_ranks(t, world)
        ap_bytes = Tpre * HKV * APPEND_BYTES_PER_TOKHEAD
        cpu_app = None
        if rank == 0 and world == 1 and not args.no_cpu:
            import numpy as np
            import oracle as O
            na = 8192                            # 1/64 of the prefill, tokens/s scale linearly
            Kh, Vh = Kp[:na].float().cpu().numpy(), Vp[:na].float().cpu().numpy()
            rkh, rvh = RK_all[0].cpu().numpy(), RV_all[0].cpu().numpy()
            fmt_h = O.PageFormat(D, BITS, G, P)
            pool_h = np.zeros((na // P, HKV, fmt_h.page_bytes), np.uint8)
            _, t_app = oracle_timed(lambda: O.quantize_append(Kh, Vh, np.arange(na), rkh, rvh, fmt_h, pool_h))
            cpu_app = {"value": na * HKV * APPEND_BYTES_PER_TOKHEAD / t_app / 1e9, "unit": "GB/s",
                       "tokens_per_s": na / t_app, "cores": cpu_threads(), "kind": "oracle",
                       "sample": f"quantize_append of {na} of the {Tpre} prefill tokens (1/64), 8 kv heads",
                       "seconds": t_app}
        extras["append"] = {
            "config": f"C2 prefill: {Tpre} tokens x {HKV} kv heads into one layer pool (per rank)",
            "tokens_per_s": Tpre * world / t * 1e3, "token_heads_per_s": Tpre * HKV * world / t * 1e3,
            "ms": t, "GBps": ap_bytes * world / t / 1e6,
            "pct_of_8TBps": ap_bytes / t / 1e6 / NOMINAL_HBM_GBS * 100,
            "roofline": {"bound": "hbm", "achieved": ap_bytes / t / 1e6, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ap_bytes / t / 1e6 / hbm_peak, "traffic": ncu_traffic(["append_tc_kernel"]),
                         "kernel": "append_tc_kernel (tcgen05 + TMA)",
                         "algorithmic_bytes_per_launch": ap_bytes, "peak_kind": peak_kind},
        }
        if cpu_app:
            extras["append"]["cpu_baseline"] = cpu_app
        # e2e: the same call with its inputs copied from pinned host memory inside the timed
        # region (a 1/8 sample of the prefill); the cache it writes stays resident on the device,
        # so nothing comes back (host <-> device copies are then PCIe-bound, not kernel-bound)
        ne = Tpre // 8
        hK, hV = Kp[:ne].cpu().pin_memory(), Vp[:ne].cpu().pin_memory()
        hS = pre_slots[:ne].cpu().pin_memory()
        dK, dV, dS = torch.empty_like(Kp[:ne]), torch.empty_like(Vp[:ne]), torch.empty_like(pre_slots[:ne])
        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for r in range(reps + 1):
            if r == 1:
                ee0.record()
            dK.copy_(hK, non_blocking=True); dV.copy_(hV, non_blocking=True); dS.copy_(hS, non_blocking=True)
            o.quantize_append(dK, dV, dS, RK_all[0], RV_all[0], pools[0])
        ee1.record(); torch.cuda.synchronize()
        te = max_over_ranks(ee0.elapsed_time(ee1) / reps, world)
        extras["append"]["e2e"] = {"value": ne * world / te * 1e3, "unit": "tokens/s",
                                   "GBps": ne * HKV * APPEND_BYTES_PER_TOKHEAD * world / te / 1e6,
                                   "h2d_bytes_per_step": (hK.numel() + hV.numel()) * 2 + hS.numel() * 8,
                                   "d2h_bytes_per_step": 0, "ms_per_step": te,
                                   "sample": f"{ne} of the {Tpre} prefill tokens per call (1/8), K, V and slots "
                                             f"copied in from pinned host memory every call"}
        del hK, hV, hS, dK, dV, dS
    del Kp, Vp

    # ---------------- decode step inputs (per layer)
    qs = [synth.torch_decode_q(gen, B_, HQ, D, dev) for _ in range(NL)]
    ks = [synth.torch_keys(gen, B_, HKV, D, dev) for _ in range(NL)]
    vs = [synth.torch_values(gen, B_, HKV, D, dev) for _ in range(NL)]
    seq_lens = torch.full((B_,), L_, dtype=torch.int32, device=dev)
    ws = torch.empty(o.attend_workspace_bytes(B_, max_pages), dtype=torch.uint8, device=dev)
    outs = [torch.empty((B_, HQ, D), dtype=torch.bfloat16, device=dev) for _ in range(NL)]

    attn_bytes = B_ * L_ * HKV * TOKHEAD_BYTES + 2 * B_ * HQ * D * 2
    app_bytes = B_ * HKV * APPEND_BYTES_PER_TOKHEAD
    step_bytes = NL * (attn_bytes + app_bytes)

    def layer(l, ev=None):
        # one Alg. 1 DecodeStep per layer: append the step's K/V row at position L-1, attend
        if ev is not None:
            ev[0].record()
        o.decode_step(qs[l], ks[l], vs[l], page_table, seq_lens, pools[l], RK_all[l], RV_all[l], ws, outs[l])
        if ev is not None:
            ev[1].record()

    for _ in range(args.warmup):
        for l in range(NL):
            layer(l)
    torch.cuda.synchronize()
    # the step (NL decode_step calls, 3 kernels each, PDL-chained) captured once in a CUDA graph
    # (SURVEY §8(d) C2); replays launch the 96 kernels without host launch overhead
    graph, graph_err = None, None
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap):
                with torch.cuda.graph(graph, stream=cap):
                    for l in range(NL):
                        layer(l)
            torch.cuda.current_stream().wait_stream(cap)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as e:                  # capture unsupported: plain stream launches
            graph, graph_err = None, str(e)

    def step():
        if graph is not None:
            graph.replay()
        else:
            for l in range(NL):
                layer(l)

    def timed_steps(fn):
        # timed region: K whole steps, events only at its two ends (per-call events would add
        # their own stream commands to the step)
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize()
        t_start.record()
        for _ in range(args.steps):
            fn()
        t_end.record()
        torch.cuda.synchronize()
        barrier(world)
        return max_over_ranks(t_start.elapsed_time(t_end), world)

    with ClockSampler(local) as clk:
        ms_total = timed_steps(step)
    ms_stream = ms_total if graph is None else timed_steps(lambda: [layer(l) for l in range(NL)])
    ms_step = ms_total / args.steps
    value = step_bytes * world * args.steps / (ms_total * 1e-3) / 1e9
    # the step is NL decode_step calls and nothing else: the average call duration over the timed
    # region is ms_step / NL.  Cross-check: the same K steps again with CUDA events around every
    # call (each event pair adds its own stream commands, ~3 µs per call)
    dec_ms = ms_step / NL
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(NL)]
           for _ in range(args.steps)]
    for s in range(args.steps):
        for l in range(NL):
            layer(l, evs[s][l])
    torch.cuda.synchronize()
    dec_ms_events = float(np.mean([a.elapsed_time(b) for st in evs for (a, b) in st]))
    dec_bytes = attn_bytes + app_bytes
    dec_gbs = dec_bytes / dec_ms / 1e6
    # attend alone (the history already holds the step's row), same pools in turn
    ea = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(NL)]
    for l in range(NL):
        o.attend(qs[l], page_table, seq_lens, pools[l], RK_all[l], RV_all[l], ws, outs[l])
    torch.cuda.synchronize()
    for l in range(NL):
        ea[l][0].record()
        o.attend(qs[l], page_table, seq_lens, pools[l], RK_all[l], RV_all[l], ws, outs[l])
        ea[l][1].record()
    torch.cuda.synchronize()
    attn_ms = float(np.mean([a.elapsed_time(b) for (a, b) in ea]))
    attn_gbs = attn_bytes / attn_ms / 1e6

    # ---------------- e2e: host-pinned inputs/outputs through the public API
    e2e = None
    if not args.no_extras:
        # every step's inputs (q, k, v of every layer: one pinned host buffer) move host -> device
        # and its outputs device -> host inside the timed region, on a copy stream: the inputs of
        # step s + 1 are copied while step s computes (two device input buffers), the outputs of
        # step s come back while step s + 1 computes (two device output buffers); the first
        # step's inputs and the last step's outputs are exposed
        n_q, n_k = qs[0].numel(), ks[0].numel()
        per_layer = n_q + 2 * n_k
        h_in = torch.cat([torch.cat([qs[l].reshape(-1), ks[l].reshape(-1), vs[l].reshape(-1)]) for l in range(NL)])
        h_in = h_in.cpu().pin_memory()
        d_in = [torch.empty_like(h_in, device=dev) for _ in range(2)]
        d_out = [torch.empty((NL, B_, HQ, D), dtype=torch.bfloat16, device=dev) for _ in range(2)]
        h_out = torch.empty((NL, B_, HQ, D), dtype=torch.bfloat16).pin_memory()
        views = [[], []]
        for i in range(2):
            for l in range(NL):
                base = l * per_layer
                views[i].append((d_in[i][base:base + n_q].view(qs[l].shape),
                                 d_in[i][base + n_q:base + n_q + n_k].view(ks[l].shape),
                                 d_in[i][base + n_q + n_k:base + per_layer].view(vs[l].shape)))
        main, cps = torch.cuda.current_stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_d2h = [torch.cuda.Event() for _ in range(2)]
        ev_out = torch.cuda.Event()

        def e2e_run(K):
            with torch.cuda.stream(cps):
                cps.wait_stream(main)
                d_in[0].copy_(h_in, non_blocking=True)
                ev_in[0].record(cps)
            for s_ in range(K):
                i = s_ % 2
                if s_ + 1 < K:
                    with torch.cuda.stream(cps):
                        if s_ >= 1:
                            cps.wait_event(ev_done[1 - i])      # step s - 1 is done with that buffer
                        d_in[1 - i].copy_(h_in, non_blocking=True)
                        ev_in[1 - i].record(cps)
                main.wait_event(ev_in[i])
                if s_ >= 2:
                    main.wait_event(ev_d2h[i])                  # step s - 2's outputs are home
                for l in range(NL):
                    dq, dk, dv = views[i][l]
                    o.decode_step(dq, dk, dv, page_table, seq_lens, pools[l], RK_all[l], RV_all[l], ws, d_out[i][l])
                ev_done[i].record(main)
                with torch.cuda.stream(cps):
                    cps.wait_event(ev_done[i])
                    h_out.copy_(d_out[i], non_blocking=True)
                    ev_d2h[i].record(cps)
            ev_out.record(cps)
            main.wait_event(ev_out)

        e2e_run(2)
        torch.cuda.synchronize(); barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        e2e_run(args.steps)
        b.record(); torch.cuda.synchronize()
        ms_e2e = max_over_ranks(a.elapsed_time(b), world)
        e2e = {"value": step_bytes * world * args.steps / (ms_e2e * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h_in.numel() * 2, "d2h_bytes_per_step": h_out.numel() * 2,
               "ms_per_step": ms_e2e / args.steps,
               "overlap": "step s + 1 inputs H2D and step s outputs D2H on a copy stream beside the compute"}

    # ---------------- C4 leg: Llama-3-70B-shaped GQA decode (g = 8), 128k context; KV heads
    # partitioned over the ranks, 4 layer pools per rank, attend only
    if not args.no_extras and not args.no_c4:
        extras["c4_decode"] = c4_leg(args, world, rank, dev, gen, RK_all, RV_all, hbm_peak, peak_kind)


    # ---------------- CPU oracle beside the GPU (rank 0, N=1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_extras and not args.no_cpu:
        import oracle as O
        fmt = O.PageFormat(D, BITS, G, P)
        b = 0
        sub = pools[0][page_table[b].long()].cpu().numpy()
        qn = qs[0][b:b + 1].float().cpu().numpy()
        rk, rv = RK_all[0].cpu().numpy(), RV_all[0].cpu().numpy()
        pt_local = np.arange(max_pages, dtype=np.int32)[None]
        (ref, _), dt = oracle_timed(lambda: O.attend(qn, pt_local, [L_], sub, rk, rv, fmt, HKV))
        samp_bytes = L_ * HKV * TOKHEAD_BYTES + 2 * HQ * D * 2
        out32 = torch.empty((B_, HQ, D), dtype=torch.float32, device=dev)     # fp32-output mode (Z25)
        o.attend(qs[0], page_table, seq_lens, pools[0], RK_all[0], RV_all[0], ws, out32)
        got = out32[b].cpu().numpy()
        cpu = {"value": samp_bytes / dt / 1e9, "unit": "GB/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": "layer 0, sequence 0, all 8 kv heads x 32768 tokens (1/16 of one layer-step)",
               "seconds": dt, "parity_max_abs_fp32_out": float(np.abs(got - ref[0]).max()),
               "parity_tolerance": 2e-3}

    if not args.no_extras and rank == 0:
        if not args.no_cpu and world == 1:
            extras["c1_end_to_end"] = c1_leg(args, dev)
        extras["c5_subset"] = c5_leg(args, dev, hbm_peak, subset=True)

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u2 codes + f16 meta, f32 accumulate", "data": "synthetic",
        "config": workload_config(args),
        "pct_of_8TBps": value / world / NOMINAL_HBM_GBS * 100,
        "roofline": {"bound": "hbm", "achieved": dec_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": dec_gbs / hbm_peak,
                     "traffic": ncu_traffic(["attend_prologue_kernel", "attend_partial_mma", "attend_merge_kernel"]),
                     "traffic_source": "profiles/ncu_traffic.json (ncu --set full, per launch)",
                     "kernel": "oscar_decode_step (prologue with append + partial + merge), one layer",
                     "algorithmic_bytes_per_launch": dec_bytes, "avg_launch_us": dec_ms * 1e3,
                     "avg_launch_us_source": "timed region / (steps x layers): the step is only decode_step calls",
                     "avg_launch_us_per_call_events": dec_ms_events * 1e3, "peak_kind": peak_kind},
        "streaming_kernel_ncu": (lambda r: None if r is None else {
            "kernel": "attend_partial_mma (85 % of the decode step)", "duration_us": r[0],
            "algorithmic_bytes": B_ * L_ * HKV * TOKHEAD_BYTES, "dram_bytes": r[1],
            "GBps": B_ * L_ * HKV * TOKHEAD_BYTES / r[0] / 1e3,
            "frac": B_ * L_ * HKV * TOKHEAD_BYTES / r[0] / 1e3 / hbm_peak,
            "source": "profiles/ncu_traffic.json: ncu --set full, serialised launch (not a bench timing)"})(
            ncu_kernel("attend_partial_mma")),
        "attend_only": {"avg_launch_us": attn_ms * 1e3, "GBps": attn_gbs, "frac": attn_gbs / hbm_peak,
                        "algorithmic_bytes_per_launch": attn_bytes,
                        "kernel": "oscar_attend (prologue + partial + merge)"},
        "gpu_launches": launches_per_layer * NL * args.steps,
        "launch_mode": "cuda_graph (one graph of the 32-layer step, replayed)" if graph is not None else
                       f"stream launches{' (graph capture failed: ' + graph_err + ')' if graph_err else ''}",
        "stream_launches": {"ms_per_step": ms_stream / args.steps,
                            "GBps": step_bytes * world * args.steps / (ms_stream * 1e-3) / 1e9},
        "clocks": clk.summary(),
        "variant": args.variant,
        "process_group": ({"backend": dist.get_backend(), "world_size": dist.get_world_size()}
                          if dist.is_initialized() else None),
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    line.update(extras)
    if rank == 0:
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
