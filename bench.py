"""Benchmark of the Cascading KV Cache hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg3|cfg2|cfg5] [--layers L] [--streams S] [--shard-of W]

One STEP = one strided prefill of the whole synthetic sequence through every layer of the
workload (Alg. 1, rows a1-a7 of SURVEY.md section 8, plus the NCCL gather of outputs a9 when
N > 1).  Default workload (configs[2]): 1M tokens through a 65K cascade cache (64 sinks,
N = 8 sub-caches, stride 4096, Llama-3-8B attention shape: 32 q-heads / 8 kv-heads, d = 128,
bf16), one layer.  --workload cfg5 (configs[4]): the same through 32 independent layers, the
layers' chunks issued chunk-major on S concurrent streams (default 4).  Each step starts from
empty caches (cascade_reset, inside the timed region).  Inputs are generated on the device
before timing (seeded per layer; when L distinct input sets do not fit in HBM the layers cycle
over as many sets as fit -- every layer still computes its own cascade); they exceed the 126 MB
L2, so no flush is needed between steps.  Row a8 (decode) is measured in the same run on
configs[3] (64 sequences x 16K cache, state from a real GPU prefill of the 128K prefix) and
reported under "decode".

N > 1 (torchrun, one process per GPU): prefill is kv-head sharded (rank r owns kv-heads
[r*Hkv/N, (r+1)*Hkv/N) and their q-heads; independent cascades) and each (layer, chunk)
output shard is all_gathered with NCCL on a side stream; decode is batch sharded (64/N
sequences per rank), its per-step outputs all_gathered the same way.  Total work is
fixed -> "scaling": "strong".  Times are the max over ranks of the device-timed K steps.

--shard-of W (N = 1): runs rank 0's shard of a W-rank job (Hq/W q-heads, Hkv/W kv-heads) on one
GPU -- the per-rank shapes of the scaling run, measured without the collective.

--impl reference times the fp64 CPU oracle (oracle/) on the host cores, rank 0 only: each step
is one steady-state chunk (the oracle's cascade filled by score injection to chunk 128) for one
q-head, scaled to the whole workload by its measured cost per (query, key) pair; the pair
count comes from the oracle's own Alg. 2 counters.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill tok/s at 1M ctx, 65K cascade cache; decode tok/s; % TC/HBM peak"

T_START = time.time()


def log(msg):
    print(f"[bench {time.time() - T_START:7.1f}s] {msg}", file=sys.stderr, flush=True)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=float(p["hbm_gbs"]), bf16=float(p["bf16_tflops"]),
                    bf16_sus=float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback (B200_PROFILING.md)")


WORKLOADS = {
    "cfg3": dict(name="cfg3_1m_65k", desc="configs[2]: Llama-3-8B attention layer, 1M-token passkey-shaped "
                 "synthetic prefill through a 65K cascade cache (64 sinks + 8 x 8192), stride 4096"),
    "cfg2": dict(name="cfg2_llama8b_4k", desc="configs[1]: Llama-3-8B attention layer, 32K prefill, "
                 "4K cascade cache (64 sinks + 4 x 1024), stride 1024"),
    "stack": dict(name="cfg5_8gpu_32l", desc="SURVEY 8(f) NEXT #4: coupled Llama-3-8B attention layers (d_model 4096, "
                  "synthetic q/k/v/o projections + residual, layer l+1 fed by layer l), 1M-token prefill through a "
                  "65K cascade cache per layer (64 sinks + 8 x 8192), stride 4096, layers as a wavefront over "
                  "per-layer streams"),
    "cfg5": dict(name="cfg5_8gpu_32l", desc="configs[4]: 32 independent Llama-3-8B attention layers, 1M-token "
                 "passkey-shaped synthetic prefill through a 65K cascade cache each (64 sinks + 8 x 8192), "
                 "stride 4096, head-sharded across the ranks"),
}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        time.sleep(0.05)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------------
# oracle legs (the reference arm and the cpu_baseline): test infrastructure, never the product
# ---------------------------------------------------------------------------------------------

def oracle_pairs(spec):
    """Visible (query, key) pairs per q-head of one layer over the whole run, from the ORACLE's
    own Alg. 2 counters (oracle.cascade.CascadeHead, payload-free tokens): sum over chunks of
    m * n_resident + m (m + 1) / 2."""
    from oracle.cascade import CascadeHead, Token
    head = CascadeHead(spec["sink_size"], spec["cache_size"], spec["num_cascades"])
    m, T = spec["stride"], spec["tokens"]
    pairs = 0
    for start in range(0, T, m):
        mm = min(m, T - start)
        pairs += mm * head.n_resident() + mm * (mm + 1) // 2
        for t in range(start, start + mm):
            head.add_token(Token(origin=t))
        head.events.clear()
    return pairs


class OracleSampler:
    """The fp64 oracle (as it stands) on one q-head / kv-head pair of the workload,
    its cascade filled to a steady-state occupancy by score injection; each sample() runs the
    oracle's strided-prefill step on the next chunk and returns (seconds, pairs)."""

    def __init__(self, spec, fill_chunks=128):
        import numpy as np
        import torch
        from oracle.model import CascadeOracle, OracleConfig
        from paper_2406_17808_b200.synth import Synth, config_seed
        self.np, self.torch = np, torch
        G = 1        # one q-head of one kv-head: the per-pair cost is what is measured (bounded sample)
        self.G, self.m = G, spec["stride"]
        fill_chunks = min(fill_chunks, spec["tokens"] // self.m - 8)
        self.orc = CascadeOracle(OracleConfig(1, 1, G, 1, spec["head_dim"], spec["sink_size"], spec["cache_size"],
                                              spec["num_cascades"], rope_theta=spec["rope_theta"],
                                              round_operands="bf16"))
        self.syn = Synth(1, G, 1, spec["head_dim"], config_seed(int(spec["key"][3])), eps=spec["eps"])
        t0 = time.perf_counter()
        S = self.orc.cfg.s_tot
        for c in range(fill_chunks):
            _, k, v = self.syn.chunk(c * self.m, self.m)
            f = k.to(torch.float64).numpy()
            s = np.zeros((1, 1, S + self.m))
            self.orc.update_with_scores(0, f, v.to(torch.float64).numpy(), s)
        self.next = fill_chunks
        self.fill_s = time.perf_counter() - t0
        self.threads = len(os.sched_getaffinity(0))

    def n_cached(self):
        return self.orc.heads[0][0][0].n_resident()

    def sample(self):
        q, k, v = self.syn.chunk(self.next * self.m, self.m)
        self.next += 1
        n_c = self.n_cached()
        pairs = self.G * (self.m * n_c + self.m * (self.m + 1) // 2)
        f = lambda t: t.to(self.torch.float64).numpy()
        q, k, v = f(q), f(k), f(v)
        t0 = time.perf_counter()
        self.orc.prefill_stride(0, q, k, v)
        return time.perf_counter() - t0, pairs


def run_reference(args, spec, wl, layers):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    total_pairs = oracle_pairs(spec) * spec["num_q_heads"] * layers
    smp = OracleSampler(spec)
    log(f"oracle filled to n_cached {smp.n_cached()} in {smp.fill_s:.1f} s")
    for _ in range(args.warmup):
        smp.sample()
    secs, pairs = 0.0, 0
    for _ in range(args.steps):
        dt, p = smp.sample()
        secs += dt
        pairs += p
    per_pair = secs / pairs
    value = spec["tokens"] / (per_pair * total_pairs)
    sample = (f"per step: one steady-state {spec['stride']}-token chunk (n_cached ~{smp.n_cached()}) of one "
              f"q-head / kv-head pair through the fp64 numpy oracle; scaled to the whole "
              f"workload ({layers} layer(s), {spec['num_q_heads']} q-heads) by its measured cost per (query, key) "
              f"pair ({per_pair * 1e9:.3f} ns/pair x {total_pairs:.3e} pairs, oracle counters)")
    line = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["desc"], "layers": layers}, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": smp.threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# GPU legs
# ---------------------------------------------------------------------------------------------

def decode_bench(args, dev, spec, peaks, world, rank, comm, use_dist):
    """configs[3]: 64 sequences, 16K cascade cache (N = 4), single-token steps (row a8).  The
    state is a real GPU prefill of each sequence's 128K-token prefix.  N > 1: the sequences are
    split across the ranks and every step's outputs all_gathered on a side stream."""
    import torch
    import torch.distributed as dist
    from paper_2406_17808_b200 import cascade as C
    from paper_2406_17808_b200.synth import Synth, config_seed
    B_all, m = spec["batch"], spec["stride"]
    if B_all % world:
        return {"error": f"{B_all} sequences do not split over {world} ranks"}
    B = B_all // world
    cfg = C.CascadeConfig(batch=B, num_q_heads=spec["num_q_heads"], num_kv_heads=spec["num_kv_heads"],
                          head_dim=spec["head_dim"], sink_size=spec["sink_size"], cache_size=spec["cache_size"],
                          num_cascades=spec["num_cascades"], max_stride=m, dtype="bf16",
                          rope_theta=spec["rope_theta"])
    cas = C.Cascade(cfg, device=dev)
    syn = Synth(B_all, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, config_seed(4), eps=spec["eps"])
    bs = slice(rank * B, (rank + 1) * B)
    t0 = time.time()
    for start in range(0, spec["tokens"], m):          # real prefill of the 128K prefix
        q, k, v = syn.chunk(start, m, device="cuda")
        cas.prefill_stride(0, q[bs].contiguous(), k[bs].contiguous(), v[bs].contiguous())
    torch.cuda.synchronize()
    log(f"decode state: real prefill of {B} x {spec['tokens']} tokens in {time.time() - t0:.1f} s")
    steps = spec["decode_steps"]
    qs, ks, vs = [], [], []
    for i in range(steps):
        q, k, v = syn.chunk(spec["tokens"] + i, 1, device="cuda")
        qs.append(q[bs, 0].contiguous()); ks.append(k[bs, 0].contiguous()); vs.append(v[bs, 0].contiguous())
    R = 4
    outs = [torch.empty_like(qs[0]) for _ in range(R)]
    gath = [torch.empty((world,) + tuple(qs[0].shape), dtype=qs[0].dtype, device="cuda") for _ in range(R)] \
        if use_dist else None
    ev_free = [None] * R
    main = torch.cuda.current_stream()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    cas.profile_enable(True)
    cas.profile_read()
    n0 = cas.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        o = outs[i % R]
        if ev_free[i % R] is not None:
            main.wait_event(ev_free[i % R])
        cas.decode(0, qs[i], ks[i], vs[i], out=o)
        if use_dist:
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)
            with torch.cuda.stream(comm):
                dist.all_gather_into_tensor(gath[i % R].view(-1), o.view(-1))
                fe = torch.cuda.Event()
                fe.record(comm)
            ev_free[i % R] = fe
    if use_dist:
        main.wait_stream(comm)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if use_dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    prof = cas.profile_read()
    st = cas.state(0)
    n_c = st["n_cached"]
    bytes_per_step = B * cfg.num_kv_heads * (n_c + 1) * (4 * cfg.head_dim + 20)
    res = {"workload": "configs[3]: 64 sequences x 128K context through a 16K cascade cache "
                       "(64 sinks + 4 x 4096), GQA 32q/8kv d=128 bf16, single-token steps; state "
                       "from a real GPU prefill of the 128K prefix (stride 4096)",
           "value": B_all * steps / (ms / 1e3), "unit": "tok/s", "steps": steps, "ms_per_step": ms / steps,
           "n_cached": n_c, "launches_per_step": (cas.launch_count() - n0) / steps,
           "parallelism": f"batch sharding x{world} ({B} sequences per rank, NCCL all_gather of every step's outputs)"
                          if use_dist else "1 GPU",
           "hbm_algorithmic_bytes_per_step_per_rank": bytes_per_step,
           "hbm_frac": bytes_per_step / (ms / steps / 1e3) / (peaks["hbm"] * 1e9)}
    res["kernels_ms_per_step"] = {k: v[0] / steps for k, v in prof.items() if v[1]}
    cas.close()
    return res


def stack_bench(args, spec, wl, peaks):
    """--workload stack: Alg. 1's layer loop over L coupled synthetic attention
    layers through cascade_stack_prefill (projections by cuBLASLt inside the library, every layer's
    attention + cache update by the cascade kernels, the layers of consecutive chunks overlapping on
    per-layer streams).  One step = the whole sequence through every layer from empty caches."""
    import torch
    from paper_2406_17808_b200 import cascade as C
    L = args.layers or 4
    Hq, Hk, d, m, T, B = (spec["num_q_heads"], spec["num_kv_heads"], spec["head_dim"], spec["stride"],
                          spec["tokens"], spec["batch"])
    D = Hq * d
    cfg = C.CascadeConfig(num_layers=L, batch=B, num_q_heads=Hq, num_kv_heads=Hk, head_dim=d,
                          sink_size=spec["sink_size"], cache_size=spec["cache_size"],
                          num_cascades=spec["num_cascades"], max_stride=m, dtype="bf16",
                          rope_theta=spec["rope_theta"])
    cas = C.Cascade(cfg)
    g = torch.Generator(device="cuda").manual_seed(5_000_000)
    sc = 1.0 / D ** 0.5
    rnd = lambda *shape: (torch.randn(shape, generator=g, device="cuda") * sc).to(torch.bfloat16)
    ws = [(rnd(D, Hq * d), rnd(D, Hk * d), rnd(D, Hk * d), rnd(Hq * d, D)) for _ in range(L)]
    st = C.Stack(cas, ws, D)
    x = torch.randn((B, T, D), generator=g, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    log(f"stack: {L} layers, inputs ready")

    def step():
        for l in range(L):
            cas.reset(l)
        st.prefill(x, m, y)

    for i in range(args.warmup):
        step()
        torch.cuda.synchronize()
        log(f"warmup step {i} done")
    clocks = ClockSampler(0)
    clocks.start()
    cas.profile_enable(True)
    cas.profile_read()
    n0 = cas.launch_count()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = cas.profile_read()
    clk = clocks.stop()
    ms_step = ms / args.steps
    useful = prof["attn_fwd"][2] / args.steps
    nchunks = (T + m - 1) // m
    gemm_flops = 2.0 * B * T * D * (Hq * d + 2 * Hk * d + Hq * d) * L
    serial = sum(v[0] for v in prof.values()) / args.steps
    res = {"metric": METRIC, "value": T * B / (ms_step / 1e3), "unit": "tok/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init projections)",
           "config": {"workload": wl["desc"], "tokens": T, "batch": B, "stride": m, "layers": L, "d_model": D,
                      "heads": f"{Hq}q/{Hk}kv d={d}", "cache": spec["cache_size"], "cascades": spec["num_cascades"],
                      "l2": "inputs and cache state exceed L2; no flush needed"},
           "stack": {"attention_useful_tflops": useful / (ms_step / 1e3) / 1e12,
                     "gemm_tflops_per_step": gemm_flops / 1e12,
                     "all_useful_tflops": (useful + gemm_flops) / (ms_step / 1e3) / 1e12,
                     "peak_sustained": peaks["bf16_sus"],
                     "cascade_kernels_ms_per_step": serial,
                     "note": "cascade_kernels_ms_per_step sums the event-timed cascade launch groups of all layer "
                             "streams (they overlap on the device, so it may exceed ms_per_step); the rest of the "
                             "step is the cuBLASLt projections"},
           "kernels": {k: {"ms_per_step": v[0] / args.steps, "launch_groups": v[1]} for k, v in prof.items() if v[1]},
           "gpu_launches": cas.launch_count() - n0, "gpu_launches_note": "cascade kernels only (+ 4 cuBLASLt GEMMs "
           f"per layer-chunk: {4 * L * nchunks * args.steps})", "clocks": clk}
    print(json.dumps(res), flush=True)
    st.close()
    cas.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=list(WORKLOADS))
    ap.add_argument("--layers", type=int, default=0, help="override the workload's layer count")
    ap.add_argument("--streams", type=int, default=0, help="concurrent layer streams (default min(L, 4))")
    ap.add_argument("--shard-of", type=int, default=1, help="N = 1: run rank 0's shard of a W-rank job")
    ap.add_argument("--tokens", type=int, default=0, help="override sequence length (debug only)")
    ap.add_argument("--score-mode", default="exact", choices=["exact", "onepass"],
                    help="per-key mass: exact two-pass (default) or the paper's one-pass estimator")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-onepass", action="store_true", help="skip the one-pass estimator line")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2406_17808_b200.synth import CONFIGS
    wl = WORKLOADS[args.workload]
    spec = dict(CONFIGS[wl["name"]], key=wl["name"])
    if args.tokens:
        spec["tokens"] = args.tokens
    L = args.layers or spec["num_layers"]
    if args.impl == "reference":
        run_reference(args, spec, wl, L)
        return
    if args.workload == "stack":
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        if int(os.environ.get("RANK", "0")) == 0:
            stack_bench(args, spec, wl, load_peaks())
        return

    import torch
    import torch.distributed as dist
    from paper_2406_17808_b200 import cascade as C
    from paper_2406_17808_b200.dist import gather_heads, shard_range
    from paper_2406_17808_b200.synth import Synth, config_seed, passkey_depth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # under torchrun (RANK set) the NCCL path runs even at world size 1 (the gathers are then
    # one-rank all_gathers: the same code path on one GPU); plain `python bench.py` has none
    use_dist = "RANK" in os.environ
    torch.cuda.set_device(local)
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = load_peaks()

    Hq, Hk, d = spec["num_q_heads"], spec["num_kv_heads"], spec["head_dim"]
    emu = args.shard_of if world == 1 else 1                # per-rank shape emulated on one GPU
    q_sl, k_sl = shard_range(rank, world * emu, Hq, Hk)     # kv-head sharding (independent heads)
    hq, hk = q_sl.stop - q_sl.start, k_sl.stop - k_sl.start
    m, T, B = spec["stride"], spec["tokens"], spec["batch"]
    nchunks = (T + m - 1) // m
    S = args.streams or min(L, 4)
    cfg = C.CascadeConfig(num_layers=L, batch=B, num_q_heads=hq, num_kv_heads=hk, head_dim=d,
                          sink_size=spec["sink_size"], cache_size=spec["cache_size"],
                          num_cascades=spec["num_cascades"], max_stride=m, dtype="bf16",
                          rope_theta=spec["rope_theta"], score_mode=args.score_mode)
    cas = C.Cascade(cfg, device=local)

    # ---- inputs, generated on the device (full heads, then this rank's shard), per layer seed ----
    set_bytes = 2 * nchunks * B * m * (hq + 2 * hk) * d
    free = torch.cuda.mem_get_info()[0]
    n_sets = max(1, min(L, int((free * 0.6) // set_bytes)))
    sets = []
    for si in range(n_sets):
        seed = config_seed(int(spec["key"][3]), si)
        syn = Synth(B, Hq, Hk, d, seed, eps=spec["eps"],
                    passkey_depth=passkey_depth(seed, T) if spec.get("passkey") else None)
        Q = torch.empty((nchunks, B, m, hq, d), dtype=torch.bfloat16, device="cuda")
        K = torch.empty((nchunks, B, m, hk, d), dtype=torch.bfloat16, device="cuda")
        V = torch.empty_like(K)
        for c in range(nchunks):
            q, k, v = syn.chunk(c * m, m, device="cuda")
            Q[c].copy_(q[:, :, q_sl])
            K[c].copy_(k[:, :, k_sl])
            V[c].copy_(v[:, :, k_sl])
        sets.append((Q, K, V))
    log(f"inputs ready: {n_sets} input set(s) for {L} layer(s), {nchunks} chunks of {m}")
    streams = [torch.cuda.current_stream()] + [torch.cuda.Stream() for _ in range(S - 1)]
    comm = torch.cuda.Stream() if use_dist else None
    R = 3                                                   # output ring per stream
    outs = [[torch.empty((B, m, hq, d), dtype=torch.bfloat16, device="cuda") for _ in range(R)] for _ in range(S)]
    gath = [[torch.empty((world, B, m, hq, d), dtype=torch.bfloat16, device="cuda") for _ in range(R)]
            for _ in range(S)] if use_dist else None
    torch.cuda.synchronize()

    ev_free = [[None] * R for _ in range(S)]   # per output slot: the gather that last read it
    slot = [0] * S

    def step():
        for l in range(L):
            cas.reset(l, stream=streams[l % S])
        for c in range(nchunks):
            for l in range(L):
                si = l % S
                st = streams[si]
                Q, K, V = sets[l % n_sets]
                r = slot[si]
                slot[si] = (r + 1) % R
                if ev_free[si][r] is not None:
                    st.wait_event(ev_free[si][r])
                o = outs[si][r]
                cas.prefill_stride(l, Q[c], K[c], V[c], out=o, stream=st)
                if use_dist:
                    ev = torch.cuda.Event()
                    ev.record(st)
                    comm.wait_event(ev)
                    with torch.cuda.stream(comm):
                        gather_heads(o, world, buf=gath[si][r], assemble=False)   # no reshape copy
                        fe = torch.cuda.Event()
                        fe.record(comm)
                    ev_free[si][r] = fe
        for st in streams[1:]:
            streams[0].wait_stream(st)
        if use_dist:
            streams[0].wait_stream(comm)

    for i in range(args.warmup):
        step()
        torch.cuda.synchronize()
        log(f"warmup step {i} done")
    if use_dist:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    cas.profile_enable(True)
    cas.profile_read()
    n0 = cas.launch_count()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    log(f"timed {args.steps} steps: {ms:.1f} ms")
    launches = cas.launch_count() - n0
    prof = cas.profile_read()
    cas.profile_enable(False)
    clk = clocks.stop()
    if use_dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = T * B / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (attention pass 1) + the others ----
    def rate(cls):
        tms, cnt, work = prof[cls]
        return (work / (tms / 1e3) if tms > 0 else 0.0), tms, cnt, work
    kern = {}
    for cls in cas.PROFILE_CLASSES:
        r, tms, cnt, work = rate(cls)
        if cnt:
            kern[cls] = {"ms_per_step": tms / args.steps, "launch_groups": cnt}
    r1, t1, c1, w1 = rate("attn_fwd")
    r2, t2, c2, w2 = rate("attn_score")
    rm, tm, cm, wm = rate("maintenance")
    concurrent = S > 1
    # the attention kernels run inside a seconds-long, power-capped step: the roofline peak is
    # the SUSTAINED bf16 figure (MEASURED_PEAKS.json bf16_tflops_sustained); burst reported beside
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            traffic = json.load(f)["attn_fwd"]["dram_bytes_per_launch"]
    except Exception:
        pass
    roof = {"kernel": "attn_fwd (pass 1: O and LSE over [sinks | cascade | chunk])", "bound": "tensor",
            "achieved": r1 / 1e12, "peak": peaks["bf16_sus"], "unit": "TFLOP/s",
            "frac": r1 / 1e12 / peaks["bf16_sus"], "frac_of_burst": r1 / 1e12 / peaks["bf16"],
            "traffic": traffic if not emu > 1 and L == 1 else None,
            "traffic_note": "dram read+write bytes of one steady-state launch, profiles/ncu_traffic_r02.json",
            "peak_source": peaks["src"] + " bf16 dense, sustained (kernel timed inside a long step)",
            "work": "4*d flops per visible (query, key) pair"}
    if concurrent:
        roof["note"] = (f"{S} concurrent layer streams: each launch's event span includes time the SMs spend on "
                        "other streams' kernels, so frac is a lower bound")
    extra_roof = {
        "attention_total": {"kernels": "attn_fwd + attn_score",
                            "achieved": w1 / ((t1 + t2) / 1e3) / 1e12 if t1 + t2 > 0 else 0,
                            "peak": peaks["bf16_sus"], "unit": "TFLOP/s",
                            "frac": (w1 / ((t1 + t2) / 1e3) / 1e12 / peaks["bf16_sus"]) if t1 + t2 > 0 else 0,
                            "frac_of_burst": (w1 / ((t1 + t2) / 1e3) / 1e12 / peaks["bf16"]) if t1 + t2 > 0 else 0},
        "maintenance": {"kernel": "maint_coop_kernel (Alg. 2 admission, selections, K/V/mu/origin moves; "
                                  "the EMA fold runs in attn_score's epilogue)",
                        "bound": "hbm", "achieved": rm / 1e9, "peak": peaks["hbm"], "unit": "GB/s",
                        "frac": rm / 1e9 / peaks["hbm"],
                        "work": "2 (2 d es + 16) bytes per row actually moved (read + write of K, V, mu, origin)",
                        "note": "each event-timed launch includes ~5 us of launch and event edge (an empty launch of "
                                "this shape measures 5.2-6.1 us, profiles/launch_edge_r01.txt); the kernel alone: "
                                "ncu gpu__time_duration 18.6 us for a steady-state launch moving 65536 rows (69.2 MB) "
                                "= 57 % of HBM (profiles/ncu_traffic_r02.json), DESIGN.md section 4"},
        "step_useful": {"achieved": w1 / args.steps / (ms_step / 1e3) / 1e12, "unit": "TFLOP/s",
                        "note": "useful attention flops per step / whole step time (every kernel, all streams)"},
    }
    share = {k: v["ms_per_step"] / ms_step for k, v in kern.items()}
    par = (f"kv-head sharding x{world} (NCCL all_gather of outputs)" if use_dist else
           (f"rank 0 of a {emu}-rank kv-head sharding, emulated on 1 GPU" if emu > 1 else "1 GPU"))
    result = {"metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
              "config": {"workload": wl["desc"], "tokens": T, "batch": B, "stride": m,
                         "cache": spec["cache_size"], "sinks": spec["sink_size"],
                         "cascades": spec["num_cascades"], "heads": f"{Hq}q/{Hk}kv d={d}",
                         "heads_per_rank": f"{hq}q/{hk}kv", "layers": L, "layer_streams": S,
                         "distinct_input_sets": n_sets, "parallelism": par, "score_mode": args.score_mode,
                         "l2": "inputs and cache state exceed L2; no flush needed"},
              "roofline": roof, "roofline_other": extra_roof, "kernels": kern, "kernel_share": share,
              "gpu_launches": launches, "clocks": clk}
    if use_dist:
        result["collective"] = {"op": "all_gather_into_tensor (NCCL) of every (layer, chunk) output shard",
                                "bytes_per_step_per_rank": 2 * B * m * hq * d * nchunks * L}

    # ---- e2e: host (pinned) buffers through cascade_prefill_stride_host_async ----
    # (every chunk's q/k/v go host->device and its output device->host inside the timed region;
    # the library overlaps those copies with the neighbouring chunks' compute)
    if not args.no_e2e:
        log("e2e start")
        Q, K, V = sets[0]
        Qh = torch.empty(Q.shape, dtype=Q.dtype, pin_memory=True)
        Kh = torch.empty(K.shape, dtype=K.dtype, pin_memory=True)
        Vh = torch.empty(V.shape, dtype=V.dtype, pin_memory=True)
        Oh = torch.empty((2 * L,) + tuple(Q.shape[1:]), dtype=Q.dtype, pin_memory=True)
        Qh.copy_(Q); Kh.copy_(K); Vh.copy_(V)
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for l in range(L):
            cas.reset(l)
        for c in range(nchunks):
            for l in range(L):
                # outputs: a ring of 2 L host slots; the library's two staging sets alternate per
                # call and a slot is reused only two calls per layer later (its copy is done)
                cas.prefill_stride_host_async(l, Qh[c], Kh[c], Vh[c], Oh[(c % 2) * L + l])
        cas.host_wait()                      # every output is in host memory
        f1.record()
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        if use_dist:
            t = torch.tensor([ems], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        per_call_in = (Q[0].numel() + K[0].numel() + V[0].numel()) * 2
        result["e2e"] = {"value": T * B / (ems / 1e3), "unit": "tok/s",
                         "h2d_bytes_per_step": per_call_in * nchunks * L * world,
                         "d2h_bytes_per_step": Q[0].numel() * 2 * nchunks * L * world,
                         "api": "cascade_prefill_stride_host_async + cascade_host_wait (pinned host q/k/v/out; "
                                "copies on library streams, overlapped with compute; layers in call order)"}
        del Qh, Kh, Vh, Oh

    # ---- the paper's one-pass estimator on the same inputs: another handle,
    # its own warm-up, the same timed-step definition; reported beside the exact-mass headline ----
    if not args.no_onepass and not use_dist and args.score_mode == "exact" and L == 1:
        log("one-pass start")
        cfg1 = C.CascadeConfig(**{**cfg.__dict__, "score_mode": "onepass"})
        cas1 = C.Cascade(cfg1, device=local)
        Q, K, V = sets[0]

        def step1():
            cas1.reset(0)
            for c in range(nchunks):
                cas1.prefill_stride(0, Q[c], K[c], V[c], out=outs[0][c % R])

        for _ in range(3):
            step1()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        for _ in range(args.steps):
            step1()
        g1.record()
        torch.cuda.synchronize()
        oms = g0.elapsed_time(g1) / args.steps
        result["onepass"] = {"value": T * B / (oms / 1e3), "unit": "tok/s", "ms_per_step": oms,
                             "score_mode": "onepass (Alg. 3 normaliser l + l rho / gamma, P:646; no pass 2)",
                             "note": "the paper's estimator instead of the exact two-pass mass (reading Q6); same "
                                     "inputs and step; DESIGN.md section 6b for its deviation from the exact mass"}
        cas1.close()

    del sets, outs, gath
    cas.close()
    torch.cuda.empty_cache()
    if not args.no_decode and emu == 1:
        log("decode start")
        try:
            result["decode"] = decode_bench(args, local, dict(CONFIGS["cfg4_decode"]), peaks, world, rank, comm, use_dist)
        except Exception as e:   # reported, never hidden
            result["decode"] = {"error": repr(e)}
    if rank == 0 and not args.no_cpu and world == 1:
        log("cpu baseline start")
        smp = OracleSampler(spec)
        secs, pairs = smp.sample()
        total_pairs = oracle_pairs(spec) * Hq * L
        per_pair = secs / pairs
        result["cpu_baseline"] = {
            "value": T * B / (per_pair * total_pairs), "unit": "tok/s", "cores": smp.threads, "kind": "oracle",
            "sample": f"one steady-state {m}-token chunk (n_cached {smp.n_cached()}) of one q-head "
                      f"({pairs:.3e} pairs) timed in {secs:.1f} s after a {smp.fill_s:.1f} s score-injection "
                      f"fill; scaled by cost per (query, key) pair to the run's {total_pairs:.3e} pairs"}
    if rank == 0:
        print(json.dumps(result), flush=True)
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
