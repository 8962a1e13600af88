"""bench.py -- effective attention TFLOP/s of the calibrated sparse attention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl csa|reference] [--config wan720]

One timed step = one calibrated sparse attention layer forward (a7 MASK heads + a8 REPETITIVE
heads) over the workload's synthetic Q/K/V, through the C ABI, with the plan produced beforehand by
the calibration path's compiler (a6) -- calibration is offline in the paper.
The calibration statistics pass (a2-a5, one prompt) and the plan compile (a6) of the same layer
are timed in the same run and reported under "phases".

value = FLOP_kept / step time, FLOP_kept = 4 d batch sum_h kept_area(h).
N > 1: heads sharded over ranks (Ulysses all-to-all of Q, K, V before and O after, NCCL), value =
all ranks' FLOP_kept / max-over-ranks step time, scaling "strong" (one layer split over N GPUs).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2603_05503_b200 import inputs, ulysses  # noqa: E402

METRIC = "effective attn TFLOP/s & % bf16 roofline, speedup vs dense, 1/2/4/8 B200"
ANCHOR_K = 5          # anchor rows of a REPETITIVE head (k of P:616-622, Table)
MAX_ABS, MEAN_ABS = 2e-2, 2e-3   # north-star tolerances (bf16 I/O, fp32 accumulation)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="csa", choices=["csa", "reference"])
    ap.add_argument("--config", default="wan720", choices=["wan480", "wan720", "mochi", "mochi85"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--rep-heads", type=int, default=4, help="REPETITIVE (anchor) heads, k=5")
    ap.add_argument("--no-extras", action="store_true", help="skip dense/SDPA/e2e/cpu legs")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--overlap-chunks", type=int, default=1,
                    help="head chunks of the exchange overlapped with the attention (N > 1); "
                         "1: no overlap (default; single-GPU NCCL check: 5 chunks cost 7.6 %% "
                         "more, the overlap pays only when the exchange crosses NVLink), 0: auto "
                         "(largest divisor of H/N up to 5)")
    ap.add_argument("--exchange", action="store_true",
                    help="run the head-sharded exchange path even at N = 1 (NCCL, one rank)")
    ap.add_argument("--fused-out", action="store_true",
                    help="exchange path with the return all-to-all fused into the attention "
                         "epilogue (csa_sparse_attn_fwd_scatter into symmetric-memory receive "
                         "buffers of every rank; SURVEY 8.6)")
    return ap.parse_args()


def peaks():
    p = {"bf16_tflops": None, "bf16_tflops_sustained": None, "hbm_gbs": None, "src": "measured"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            m = json.load(fh)
        p.update({k: m.get(k) for k in ("bf16_tflops", "bf16_tflops_sustained", "hbm_gbs")})
    except OSError:
        p.update({"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                  "src": "fallback (B200_PROFILING.md)"})
    return p


def mufu_peak():
    """Measured MUFU ex2/s of the whole GPU under load (profiles/mufu_peak_b200.json, written by
    scripts/mufu_peak.cu); fallback: 16 ex2/clk/SM x 148 SMs x 1965 MHz (B200_PROFILING.md max
    clock), stated as such."""
    try:
        with open(os.path.join(ROOT, "profiles", "mufu_peak_b200.json")) as fh:
            m = json.load(fh)
        return {"ex2_per_s": float(m["ex2_per_s"]),
                "src": f"measured (profiles/mufu_peak_b200.json, {m.get('sm_mhz_last')} MHz)"}
    except (OSError, KeyError, ValueError):
        return {"ex2_per_s": 16.0 * 148 * 1965e6, "src": "16 ex2/clk/SM x 148 x 1965 MHz"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def kept_area_host(masks: np.ndarray, lay: inputs.Layout) -> np.ndarray:
    sizes = np.array([lay.block_size(c) for c in range(lay.NB)], np.int64)
    return np.einsum("hrc,r,c->h", masks.astype(np.int64), sizes, sizes)


def workload(cfg, args, heads_lo, heads_hi, rank_dev):
    """Plan inputs for all heads: keep counts + min_count for the compiler (a6), the resulting
    MASK-head masks (host, for FLOP accounting and the oracle sample), the REPETITIVE heads.

    Configs with a BASELINE sparsity (Wan 480p / 720p): generator S masks at that sparsity,
    counts = 64 * M, min_count 32.  Configs without one (Mochi, M4): the
    calibration path itself -- |D| = 8 generator-G prompts through csa_calib_accumulate at
    t = 32 of T = 64 (eps from Eq. eq:epsilon_schedule), rho = 0.5 -> min_count 4."""
    lay = cfg.layout
    rep = set(np.linspace(0, cfg.heads - 1, args.rep_heads).astype(int).tolist()) if args.rep_heads else set()
    if cfg.sparsity is not None:
        # The BASELINE sparsity is the layer's TOTAL (P:680 / P:688 count the repetition heads'
        # anchor-only area too, reading Q19): the MASK heads' generator-S target is set so that
        # sum(MASK kept areas) + |rep| * F k W N = (1 - sparsity) H N^2, i.e. every anchor head
        # keeps k / H_rows of its dense area.
        mask_heads = [h for h in range(cfg.heads) if h not in rep]
        rep_kept = ANCHOR_K / lay.H
        mask_kept = ((1.0 - cfg.sparsity) * cfg.heads - len(rep) * rep_kept) / len(mask_heads)
        mm = inputs.synthetic_masks(lay, len(mask_heads), 1.0 - mask_kept, seed=0)
        masks = np.ones((cfg.heads, lay.NB, lay.NB), np.uint8)   # REPETITIVE cells: unused
        masks[mask_heads] = mm
        counts = masks.astype(np.uint16) * np.uint16(64)
        return lay, masks, rep, counts, 32, None
    from paper_2603_05503_b200 import csa

    n_prompts, t, T = 8, 32, 64
    a_n = 0.796 + 1.41e-6 * lay.N                       # A(N)
    eps = a_n + (0.99 - a_n) * math.exp(-16.0 * t / T)  # Eq. eq:epsilon_schedule, C = 0.99, k = 16
    alphas = np.linspace(0.8, 1.6, cfg.heads)           # peak-logit scale spread across heads
    counts_t = torch.zeros(cfg.heads * lay.NB * lay.NB, dtype=torch.int16,
                           device=rank_dev).view(torch.uint16)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim_sum = torch.zeros(cfg.heads, dtype=torch.float64, device=rank_dev)
    for p in range(n_prompts):
        qc, kc, _ = inputs.structured_qk(lay, cfg.heads, cfg.d, head_seed=1, prompt_seed=p,
                                         alpha=alphas, repetitive=tuple(sorted(rep)),
                                         device=rank_dev)
        csa.calib_accumulate_sim(lay, qc, kc, eps, counts_t, 5, sim_sum)  # a2-a5 + f1, one pass
        del qc, kc
    torch.cuda.synchronize()
    calib_s = time.perf_counter() - t0
    s_head = (sim_sum / (lay.F * lay.H * n_prompts)).cpu().numpy()
    # REPETITIVE where s > gamma = 0.87 (strict, Q8): the decision is the data's,
    # not the generator's labels (which are only reported next to it)
    detected = {h for h in range(cfg.heads) if s_head[h] > 0.87}
    counts = counts_t.view(torch.int16).cpu().numpy().view(np.uint16).reshape(
        cfg.heads, lay.NB, lay.NB)
    min_count = math.ceil(0.5 * n_prompts)
    masks = np.zeros((cfg.heads, lay.NB, lay.NB), np.uint8)
    plan = csa.compile_plan(lay, counts_t, min_count)   # MASK view of every head, for accounting
    bits = plan.mask_bits.cpu().numpy().view(np.uint32)
    w32 = (lay.NB + 31) // 32
    unpacked = np.unpackbits(bits.view(np.uint8), bitorder="little").reshape(
        cfg.heads, lay.NB, w32 * 32)[:, :, :lay.NB]
    masks[:] = unpacked
    calib = {"prompts": n_prompts, "t": t, "T": T, "eps": round(eps, 6), "min_count": min_count,
             "wall_s_incl_generator": round(calib_s, 3),
             "similarity": [round(float(x), 4) for x in s_head], "gamma": 0.87,
             "repetitive_detected": sorted(detected),
             "repetitive_generated": sorted(rep)}
    return lay, masks, detected, counts, min_count, calib


def arm_config(cfg, batch, kept_fraction, rep, world):
    """The workload description both arms print (the driver compares lines with equal config)."""
    lay, H, d = cfg.layout, cfg.heads, cfg.d
    return {"workload": f"{cfg.name} single attention layer",
            "F_H_W": [lay.F, lay.H, lay.W], "tokens": lay.N, "heads": H, "head_dim": d,
            "block": lay.B, "batch": batch, "kept_fraction": round(kept_fraction, 4),
            "mask_sparsity_target": cfg.sparsity, "repetitive_heads": sorted(rep),
            "anchor_k": 5, "parallelism": f"heads{world} (Ulysses a2a)" if world > 1 else "1 GPU",
            "l2": "inputs 3x%.2f GB > 126 MB L2; no flush" % (batch * lay.N * H * d * 2 / 1e9)}


def flops_of(lay, masks, rep, heads, d, batch, anchor_k=5):
    area = kept_area_host(masks, lay)
    tot = 0
    for h in heads:
        tot += (lay.F * anchor_k * lay.W * lay.N) if h in rep else int(area[h])
    return 4.0 * d * batch * tot, tot


def time_loop(fn, steps, warmup, stream):
    """W untimed warm-ups, then K steps bracketed by (barrier +) synchronize on both sides, CUDA
    events on `stream` around the whole region and around every step.  Returns (total ms, per-step
    ms list, the last step's return value -- the timed output the parity gate checks)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    per = []
    last = None
    start.record(stream)
    for _ in range(steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        last = fn()
        e1.record(stream)
        per.append((e0, e1))
    end.record(stream)
    torch.cuda.synchronize()
    if torch.distributed.is_initialized():
        torch.distributed.barrier()
    total = start.elapsed_time(end)
    return total, [a.elapsed_time(b) for a, b in per], last


def pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, max(0, int(round(p / 100.0 * (len(xs) - 1)))))]


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"host_cores": os.cpu_count() or 1,
            "host_cores_usable": len(os.sched_getaffinity(0)), "cpu_model": model}


class OracleHeads:
    """fp64 host copies of single heads of Q, K, V (the oracle's inputs: the same bf16 values
    the GPU reads, widened exactly)."""

    def __init__(self, q, k, v):
        self.t = (q, k, v)
        self.cache = {}

    def __call__(self, h):
        if h not in self.cache:
            self.cache[h] = tuple(x[0, :, h].double().cpu().numpy() for x in self.t)
        return self.cache[h]


def oracle_unit(lay, heads64, masks, rep, h, rows, d):
    """Oracle output rows [r0, r1) of head h (MASK: masked softmax over the kept blocks, P:647-653;
    REPETITIVE: anchor-row attention + broadcast) and the unit's kept FLOPs."""
    import oracle

    qh, kh, vh = heads64(h)
    scale = 1.0 / math.sqrt(d)
    if h in rep:
        out, _ = oracle.anchor_attention_rows(lay.F, lay.H, lay.W, qh, kh, vh, scale, ANCHOR_K, rows)
        return out, 4.0 * d * (rows[1] - rows[0]) * lay.N * ANCHOR_K / lay.H
    out, _ = oracle.masked_attention_rows(qh, kh, vh, scale, lay.B, masks[h], rows)
    sizes = np.array([lay.block_size(c) for c in range(lay.NB)], np.int64)
    r = rows[0] // lay.B
    return out, 4.0 * d * (rows[1] - rows[0]) * float(masks[h, r].astype(np.int64) @ sizes)


def parity_units(lay, masks, rep, heads, seed, n_random=8, row_range=None):
    """Sampled (head, rows) units of a launch: per sampled MASK head the rows of its emptiest,
    median and fullest query block, block 0 and the ragged last block; REPETITIVE heads' first
    and last block (the broadcast rows); plus random blocks.  row_range restricts rows to a
    token shard (multi-GPU: the rank's sequence shard)."""
    rng = np.random.default_rng(seed)
    lo, hi = (0, lay.N) if row_range is None else row_range
    blocks = [r for r in range(lay.NB) if r * lay.B < hi and min((r + 1) * lay.B, lay.N) > lo]
    mask_heads = [h for h in heads if h not in rep]
    rep_heads = [h for h in heads if h in rep]
    units = set()
    for h in (mask_heads[:1] + mask_heads[-1:] + list(rng.choice(mask_heads, 2))):
        h = int(h)
        nnz = masks[h][blocks].sum(axis=1)
        order = np.argsort(nnz, kind="stable")
        for r in {blocks[order[0]], blocks[order[len(order) // 2]], blocks[order[-1]],
                  blocks[0], blocks[-1]}:
            units.add((h, r))
    for h in rep_heads[:2]:
        units.add((h, blocks[0]))
        units.add((h, blocks[-1]))
    for _ in range(n_random):
        units.add((int(rng.choice(list(heads))), int(rng.choice(blocks))))
    return [(h, (max(r * lay.B, lo), min((r + 1) * lay.B, lay.N, hi))) for h, r in sorted(units)]


def run_oracle(units, fn, threads):
    """fn(unit) on a host thread pool (the C oracle releases the GIL).  Returns (results, wall s)."""
    import concurrent.futures

    t0 = time.perf_counter()
    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(fn, units))
    return res, time.perf_counter() - t0


def parity_stats(got_rows, ref_rows):
    """(max |dO|, sum |dO|, count) over compared elements."""
    mx, sm, cnt = 0.0, 0.0, 0
    for g, r in zip(got_rows, ref_rows):
        e = np.abs(g - r)
        mx = max(mx, float(e.max()))
        sm += float(e.sum())
        cnt += e.size
    return mx, sm, cnt


def parity_record(mx, sm, cnt, n_units, where):
    mean = sm / max(cnt, 1)
    return {"max_abs": mx, "mean_abs": mean, "units": n_units, "elements": cnt,
            "tol": {"max_abs": MAX_ABS, "mean_abs": MEAN_ABS},
            "pass": bool(mx <= MAX_ABS and mean <= MEAN_ABS), "checked": where}


def cpu_oracle_sample(lay, cfg, masks, rep, heads64, seconds_target=12.0, extra_units=()):
    """The fp64 oracle, as it stands, on a bounded sample of (head, query-block) units of the same
    workload (~seconds_target of host wall time), one host thread per unit.  extra_units are
    computed in the same pool (the parity units); returns (cpu_baseline dict, their outputs)."""
    threads = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)
    mask_heads = [h for h in range(cfg.heads) if h not in rep]
    probe = (mask_heads[0], (lay.NB // 2 * lay.B, lay.NB // 2 * lay.B + lay.B))
    t0 = time.perf_counter()
    oracle_unit(lay, heads64, masks, rep, probe[0], probe[1], cfg.d)
    t_probe = time.perf_counter() - t0
    n_units = int(seconds_target / max(t_probe, 1e-3)) * threads
    n_units = max(threads, min(n_units, 4 * threads) - len(extra_units))
    units = list(extra_units)
    for _ in range(n_units):
        h = int(rng.choice(mask_heads))
        r = int(rng.integers(lay.NB))
        units.append((h, (r * lay.B, min((r + 1) * lay.B, lay.N))))
    for h in {u[0] for u in units}:
        heads64(h)
    res, wall = run_oracle(units, lambda u: oracle_unit(lay, heads64, masks, rep, u[0], u[1], cfg.d),
                           threads)
    flops = sum(f for _, f in res)
    return ({"value": flops / wall / 1e12, "unit": "TFLOP/s", "cores": threads, **host_info(),
             "kind": "oracle",
             "sample": f"{len(units)} (head, query-block) units of {cfg.name} ({len(extra_units)} "
                       f"stratified parity units incl. anchor heads and the ragged last block, "
                       f"the rest random MASK blocks; 128 query rows each, kept keys only), fp64 C "
                       f"oracle, {threads} host threads, {wall:.1f} s wall; value = sampled kept "
                       f"FLOP / wall"},
            [o for o, _ in res[:len(extra_units)]])


def relaunch(args):
    """`bench.py --gpus N` (N > 1) started without torchrun: re-exec under torch.distributed.run
    with one rank per GPU, or fail loudly when fewer than N GPUs are visible."""
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {n_dev} CUDA device(s) visible; "
                         f"refusing to report a smaller job")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl != "reference" and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    cfg = inputs.CONFIGS[args.config]
    lay = cfg.layout

    if args.impl == "reference":
        return reference_arm(args, cfg, world, rank)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    elif args.exchange or args.fused_out:  # single-rank NCCL group: the exchange path, 1 GPU
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        torch.distributed.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}",
                                             rank=0, world_size=1, device_id=dev)
    exchange = world > 1 or args.exchange or args.fused_out
    from paper_2603_05503_b200 import csa

    stream = torch.cuda.current_stream()
    H, d, B = cfg.heads, cfg.d, args.batch
    if H % world or lay.N % world:
        raise SystemExit(f"heads {H} / tokens {lay.N} not divisible by {world}")
    hp = H // world
    h_lo, h_hi = rank * hp, (rank + 1) * hp
    lay, masks, rep, counts_all, min_count, calib = workload(cfg, args, 0, H, dev)
    # head order of the exchange: LPT over the heads' kept areas (ulysses.balance_heads; a model
    # folds it into its projections), so every rank gets H/P heads of near-equal total work
    head_cost = [flops_of(lay, masks, rep, [h], d, 1)[1] for h in range(H)]
    perm = list(range(H)) if world == 1 else ulysses.balance_heads(head_cost, world)
    my_heads = perm[h_lo:h_hi]

    # ---- plan for this rank's heads (a6 through the C ABI), REPETITIVE via similarity > gamma
    counts_np = np.ascontiguousarray(counts_all[my_heads], dtype=np.uint16)
    counts = torch.from_numpy(counts_np.reshape(-1).view(np.int16)).to(dev).view(torch.uint16)
    sim = torch.tensor([calib["similarity"][h] if calib is not None else (1.0 if h in rep else 0.0)
                        for h in my_heads], dtype=torch.float64, device=dev)
    plan = csa.compile_plan(lay, counts, min_count, similarity=sim, gamma=0.87, anchor_k=ANCHOR_K)
    work = csa.build_work_list(plan, 0, hp, order=csa.default_order(lay, d))
    torch.cuda.synchronize()
    flop_rank, _ = flops_of(lay, masks, rep, my_heads, d, B)
    flop_all, area_all = flops_of(lay, masks, rep, range(H), d, B)
    dense_flop = 4.0 * d * B * H * float(lay.N) ** 2
    kept_fraction = area_all / (H * float(lay.N) ** 2)

    # ---- inputs: full-sequence tensors generated identically on every rank, then sliced
    q, k, v = inputs.qkv(B, lay.N, H, d, seed=11, device=dev)
    out = torch.empty((B, lay.N, hp, d), dtype=torch.bfloat16, device=dev)
    heads64 = OracleHeads(q, k, v)

    chunks = args.overlap_chunks or max(c for c in range(1, 6) if hp % c == 0)
    if not exchange:
        def step():
            return csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
        units = parity_units(lay, masks, rep, list(range(H)), seed=rank)
    else:
        # kernel-only reference for the roofline: this rank's heads, full sequence
        qh0, kh0, vh0 = (t[:, :, my_heads].contiguous() for t in (q, k, v))
        ql, kl, vl = (ulysses.sequence_shard(t[:, :, perm], world, rank) for t in (q, k, v))
        n_loc = lay.N // world
        units = parity_units(lay, masks, rep, list(range(H)), seed=rank, n_random=2,
                             row_range=(rank * n_loc, (rank + 1) * n_loc))
        for h in {u[0] for u in units}:
            heads64(h)            # host copies before the full tensors are dropped
        del q, k, v
        q = k = v = None

        def run_heads(qh, kh, vh, o=None):
            return csa.sparse_attn_fwd(qh, kh, vh, plan, work, out=out if o is None else o)

        hc = hp // chunks
        works = [csa.build_work_list(plan, c * hc, hc, order=csa.default_order(lay, d))
                 for c in range(chunks)]

        def run_chunk(c, qh, kh, vh, o):  # heads c*hc .. of this rank: cells c*hc ..
            return csa.sparse_attn_fwd(qh, kh, vh, plan, works[c], cell_base=c * hc, out=o)

        def run_scatter(qh, kh, vh, ptrs, recv):
            csa.sparse_attn_fwd_scatter(qh, kh, vh, plan, work, ptrs, recv)

        def layer_step(a, b_, c_):
            if args.fused_out:
                return ulysses.make_layer_step_fused_out(a, b_, c_, world, run_scatter)
            if chunks == 1:
                return ulysses.make_layer_step(a, b_, c_, world, run_heads)
            return ulysses.make_layer_step_chunked(a, b_, c_, world, run_chunk, chunks)
        step = layer_step(ql, kl, vl)

    with ClockSampler(local) as clk:
        total_ms, per, last = time_loop(step, args.steps, args.warmup, stream)
    ms = total_ms / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if exchange:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = flop_all / (ms * 1e-3) / 1e12

    # ---- parity gate on the TIMED output (the last timed step's result), sampled units
    if exchange:
        # last: this rank's [B, N/P, H, d] sequence shard, head positions in perm order
        n_loc = lay.N // world
        got = [last[0, r0 - rank * n_loc:r1 - rank * n_loc, perm.index(h)].double().cpu().numpy()
               for h, (r0, r1) in units]
        refs, _ = run_oracle(units, lambda u: oracle_unit(lay, heads64, masks, rep, u[0], u[1], d)[0],
                             len(os.sched_getaffinity(0)))
        mx, sm, cnt = parity_stats(got, refs)
        st = torch.tensor([mx, sm, cnt, len(units)], device=dev, dtype=torch.float64)
        mx_t, rest = st[:1].clone(), st[1:].clone()
        torch.distributed.all_reduce(mx_t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(rest, op=torch.distributed.ReduceOp.SUM)
        parity = parity_record(float(mx_t), float(rest[0]), int(rest[1]), int(rest[2]),
                               "every rank's sequence shard of the timed output vs fp64 oracle")
        cpu_base = None
    else:
        got = [last[0, r0:r1, h].double().cpu().numpy() for h, (r0, r1) in units]
        cpu_base, refs = (None, None)
        if rank == 0 and not args.no_extras:
            cpu_base, refs = cpu_oracle_sample(lay, cfg, masks, rep, heads64, extra_units=units)
        else:
            refs, _ = run_oracle(units,
                                 lambda u: oracle_unit(lay, heads64, masks, rep, u[0], u[1], d)[0],
                                 len(os.sched_getaffinity(0)))
        parity = parity_record(*parity_stats(got, refs), len(units),
                               "timed output vs fp64 oracle")

    pk = peaks()
    per_ms = sorted(per)
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic (seeded N(0,1) bf16 Q/K/V; generator-S calibrated-like block masks)"
                 if calib is None else
                 "synthetic (seeded N(0,1) bf16 Q/K/V; plan calibrated by this repo's a2-a6 path "
                 "on 8 generator-G prompts)"),
        "config": arm_config(cfg, B, kept_fraction, rep, world),
        "t_ms": {"median": round(statistics.median(per_ms), 4), "p10": round(pct(per_ms, 10), 4),
                 "p90": round(pct(per_ms, 90), 4), "rank": rank},
        "parity": parity,
        "gpu_launches": args.steps * launches_per_call(lay, d) * (chunks if exchange else 1),
        **({"calibration": calib} if calib is not None else {}),
        "clocks": clk.summary(),
    }
    if exchange:
        result["config"]["exchange_overlap_chunks"] = chunks
        result["config"]["exchange"] = (
            "stacked QKV all_to_all_single; O rows stored by the attention epilogue straight into "
            "every rank's symmetric-memory receive buffer (return all-to-all fused)"
            if args.fused_out else "stacked QKV all_to_all_single (1 per chunk) + O return")
        # roofline of the attention kernel on this rank (launches alone, no exchange), the
        # slowest rank's: achieved = its kept FLOPs / its mean launch time
        _, per_k, _ = time_loop(lambda: run_heads(qh0, kh0, vh0), args.steps, 2, stream)
        ms_k = statistics.mean(per_k)
        mk = torch.tensor([ms_k, flop_rank, -ms_k], device=dev, dtype=torch.float64)
        gathered = [torch.zeros_like(mk) for _ in range(world)]
        torch.distributed.all_gather(gathered, mk)
        slow = max(gathered, key=lambda t: float(t[0]))
        ach = float(slow[1]) / (float(slow[0]) * 1e-3) / 1e12
        result["roofline"] = {"bound": "tensor", "achieved": round(ach, 2),
                              "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                              "frac": round(ach / pk["bf16_tflops"], 4), "traffic": None,
                              "peak_src": f"{pk['src']} bf16 burst",
                              "kernel": attention_kernel_name(lay, cfg.d) + ", slowest rank",
                              "algorithmic_flop_per_launch": float(slow[1]),
                              "kernel_ms_per_rank": [round(float(t[0]), 3) for t in gathered],
                              "step_ms_vs_kernel_ms": round(ms / float(slow[0]), 4)}
        # e2e at N GPUs through the public API: every step copies this rank's sequence shard of
        # Q, K, V in from pinned host memory, runs the head-sharded layer (a2a, attention, a2a)
        # and copies the rank's output shard back; max over ranks.  Bytes are whole-job totals.
        hq, hk, hv = (t.cpu().pin_memory() for t in (ql, kl, vl))
        dq, dk, dv = (torch.empty_like(t) for t in (ql, kl, vl))
        step_e2e = layer_step(dq, dk, dv)
        ho = torch.empty(ql.shape, dtype=ql.dtype).pin_memory()

        def e2e_step():
            dq.copy_(hq, non_blocking=True)
            dk.copy_(hk, non_blocking=True)
            dv.copy_(hv, non_blocking=True)
            ho.copy_(step_e2e(), non_blocking=True)

        n_e2e = max(2, args.steps // 3)
        t_e2e, _, _ = time_loop(e2e_step, n_e2e, 1, stream)
        te = torch.tensor([t_e2e / n_e2e], device=dev)
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(te.item())
        result["e2e"] = {"value": round(flop_all / (t_e2e * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                         "ms_per_step": round(t_e2e, 3),
                         "h2d_bytes_per_step": 3 * ql.numel() * 2 * world,
                         "d2h_bytes_per_step": ql.numel() * 2 * world}
    if rank == 0 and not exchange and not args.no_extras:
        extras(result, args, cfg, lay, masks, rep, plan, work, q, k, v, out, flop_all, dense_flop,
               kept_fraction, per, pk, stream, dev, csa)
        result["cpu_baseline"] = dict(cpu_base)
        # extrapolated, not measured: the whole layer's kept FLOPs at the sampled rate
        result["cpu_baseline"]["extrapolated_layer_s_all_threads"] = round(
            flop_all / (cpu_base["value"] * 1e12), 1)
    if rank == 0:
        if not parity["pass"]:  # a perf number without passing parity is not reported
            result["value"] = None
            result["parity_failed"] = True
        line = json.dumps(result)
        print(line, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as fh:
                fh.write(line + "\n")
    if exchange:
        torch.distributed.destroy_process_group()
    if not parity["pass"]:
        sys.exit(3)


def attention_kernel_name(lay, d):
    """The kernel csa_sparse_attn_fwd runs for this shape (api.cu dispatch)."""
    if lay.B == 128 and lay.Bkv == 128:
        return "sparse_attn_sepp_kernel (attn5.cu)"
    if lay.B == 128:
        return f"sparse_attn_rect_kernel<{lay.Bkv},{d}> (attn_rect.cu)"
    return f"sparse_attn_kernel<{lay.B},{d}> (attn.cu)"


def launches_per_call(lay, d):
    """Our kernels per csa_sparse_attn_fwd call: at block 128 the fixed-reference kernel is
    followed by the two exact-max passes over its (normally empty) fallback list."""
    return 3 if lay.B == 128 else 1


def extras(result, args, cfg, lay, masks, rep, plan, work, q, k, v, out, flop_all, dense_flop,
           kept_fraction, per, pk, stream, dev, csa):
    ms_kernel = statistics.mean(per)
    achieved = flop_all / (ms_kernel * 1e-3) / 1e12
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_{cfg.name}_attn.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except OSError:
        pass
    result["roofline"] = {"bound": "tensor", "achieved": round(achieved, 2),
                          "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                          "frac": round(achieved / pk["bf16_tflops"], 4), "traffic": traffic,
                          "peak_src": f"{pk['src']} bf16 burst",
                          "frac_of_sustained": round(achieved / pk["bf16_tflops_sustained"], 4),
                          "kernel": attention_kernel_name(lay, cfg.d),
                          "algorithmic_flop_per_launch": flop_all}
    # ---- same-box context: cuBLAS bf16 GEMM burst on THIS box right now (the pool's
    # MEASURED_PEAKS figure stays the roofline peak; boxes differ by several percent)
    try:
        ga = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        gb = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
        best = None
        for _ in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            torch.matmul(ga, gb)
            e1.record(stream)
            e1.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        gemm = 2.0 * 8192 ** 3 / (best * 1e-3) / 1e12
        result["roofline"]["same_box_bf16_gemm_tflops"] = round(gemm, 1)
        result["roofline"]["frac_of_same_box_gemm"] = round(result["roofline"]["achieved"] / gemm, 4)
        del ga, gb
    except Exception as e:  # context only
        result["roofline"]["same_box_bf16_gemm_tflops"] = f"unavailable: {e}"
    # ---- dense comparators: our kernel on an all-ones plan, and torch SDPA (cuDNN/flash)
    H, d, B = cfg.heads, cfg.d, args.batch
    ones = torch.full((H * lay.NB * lay.NB,), 64, dtype=torch.int16, device=dev).view(torch.uint16)
    plan1 = csa.compile_plan(lay, ones, 32)
    work1 = csa.build_work_list(plan1, 0, H, order=csa.default_order(lay, d))
    t_dense, _, _ = time_loop(lambda: csa.sparse_attn_fwd(q, k, v, plan1, work1, out=out),
                              max(2, args.steps // 3), 2, stream)
    t_dense /= max(2, args.steps // 3)
    sdpa_ms = None
    try:
        qt, kt, vt = (t.transpose(1, 2) for t in (q, k, v))
        f = lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)
        t_s, _, _ = time_loop(f, 2, 1, stream)
        sdpa_ms = t_s / 2
    except Exception as e:  # library comparator only
        sdpa_ms = f"unavailable: {e}"
    ms = result["ms_per_step"]
    result["dense"] = {
        "ours_all_ones_ms": round(t_dense, 3),
        "ours_dense_tflops": round(dense_flop / (t_dense * 1e-3) / 1e12, 1),
        "torch_sdpa_ms": sdpa_ms if isinstance(sdpa_ms, str) else round(sdpa_ms, 3),
        "speedup_vs_ours_dense": round(t_dense / ms, 3),
        "speedup_vs_sdpa": None if isinstance(sdpa_ms, str) else round(sdpa_ms / ms, 3),
        "proportionality": round(t_dense / ms * kept_fraction, 3),
        "dense_equiv_tflops": round(dense_flop / (ms * 1e-3) / 1e12, 1),
    }
    # ---- phases of the whole hot path on the same layer: calibration (a2-a5) + compile (a6)
    ph = {"attn_ms": ms}
    counts_c = torch.zeros(H * lay.NB * lay.NB, dtype=torch.int16, device=dev).view(torch.uint16)
    # eps(t=25 of T=50) from Eq. eq:epsilon_schedule with A(N), host fp64
    eps = 0.796 + 1.41e-6 * lay.N + (0.99 - (0.796 + 1.41e-6 * lay.N)) * math.exp(-16 * 25 / 50)
    t_cal, _, _ = time_loop(lambda: csa.calib_accumulate(lay, q[:1], k[:1], eps, counts_c), 1, 1,
                            stream)
    t_cal2, _, _ = time_loop(lambda: csa.calib_accumulate(lay, q[:1], k[:1], eps, counts_c,
                                                       single_pass=False), 1, 1, stream)
    lse_c = torch.empty(H * lay.N, dtype=torch.float32, device=dev)
    csa.calib_accumulate(lay, q[:1], k[:1], eps, counts_c, lse_out=lse_c)
    sim_c = torch.zeros(H, dtype=torch.float64, device=dev)
    t_sim, _, _ = time_loop(lambda: csa.spatial_similarity(lay, q[:1], k[:1], lse_c, 5, sim_c), 1, 1,
                         stream)
    sim_f = torch.zeros(H, dtype=torch.float64, device=dev)
    t_fused, _, _ = time_loop(lambda: csa.calib_accumulate_sim(lay, q[:1], k[:1], eps, counts_c, 5,
                                                               sim_f), 1, 1, stream)
    ph["calib_sim_fused_ms"] = round(t_fused, 3)           # a2-a5 + f1 in one pass (2 exps/score)
    ph["calib_sim_fused_exp_frac_of_mufu"] = None          # filled below
    ph["calib_plus_sim_two_calls_ms"] = round(t_cal + t_sim, 3)
    ph["spatial_similarity_ms"] = round(t_sim, 3)          # f1: 2 exps per score
    ph["calib_accumulate_ms"] = round(t_cal, 3)             # single exponential pass (scratch)
    ph["calib_accumulate_two_pass_ms"] = round(t_cal2, 3)   # LSE pass + E pass
    calib_exps = 1.0 * H * float(lay.N) ** 2                 # one exp per score
    ph["calib_exp_per_s"] = calib_exps / (t_cal * 1e-3)
    ph["calib_qk_tflops"] = round(2.0 * d * H * float(lay.N) ** 2 / (t_cal * 1e-3) / 1e12, 1)
    # exp roofline of a2-a3: the MEASURED MUFU ex2 throughput of this pool's B200s
    # under load (scripts/mufu_peak.cu -> profiles/mufu_peak_b200.json: 16 ex2 / clk / SM at the
    # sustained clock), a fixed denominator for every run
    mufu = mufu_peak()
    ph["calib_mufu_peak_exp_per_s"] = mufu["ex2_per_s"]
    ph["calib_mufu_peak_src"] = mufu["src"]
    ph["calib_exp_frac_of_mufu"] = round(ph["calib_exp_per_s"] / mufu["ex2_per_s"], 4)
    ph["calib_sim_fused_exp_frac_of_mufu"] = round(2.0 * calib_exps / (t_fused * 1e-3)
                                                   / mufu["ex2_per_s"], 4)
    cnt = torch.from_numpy((masks.astype(np.uint16) * np.uint16(64)).reshape(-1).view(np.int16)).to(dev).view(torch.uint16)
    sim = torch.tensor([1.0 if h in rep else 0.0 for h in range(H)], dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    csa.compile_plan(lay, cnt, 32, similarity=sim, gamma=0.87, anchor_k=5)
    torch.cuda.synchronize()
    ph["compile_plan_ms_incl_readback"] = round((time.perf_counter() - t0) * 1e3, 3)
    ph["plan_bytes"] = plan.nbytes()
    # the same plan in the intervals-only form (no CSR index; the kernel walks the 1-D skip
    # list): its bytes and its attention launch, bitwise the same output
    plan_iv = csa.compile_plan(lay, cnt, 32, similarity=sim, gamma=0.87, anchor_k=5, csr=False)
    work_iv = csa.build_work_list(plan_iv, 0, H, order=csa.default_order(lay, d))
    if q.shape[2] == H:  # single-GPU layout (the exchange path holds rank-local views)
        out_iv = torch.empty_like(out)
        # alternating A/B (CSR plan, intervals-only plan) so both see the same clocks
        reps = max(2, args.steps // 2)
        t_cs, t_ivs = [], []
        for _ in range(3):
            t_a, _, _ = time_loop(lambda: csa.sparse_attn_fwd(q, k, v, plan, work, out=out_iv),
                                  reps, 1, stream)
            t_b, _, _ = time_loop(lambda: csa.sparse_attn_fwd(q, k, v, plan_iv, work_iv,
                                                              out=out_iv), reps, 1, stream)
            t_cs.append(t_a / reps)
            t_ivs.append(t_b / reps)
        ph["attn_ms_csr_plan_alternating"] = round(statistics.median(t_cs), 3)
        ph["attn_ms_intervals_only_plan"] = round(statistics.median(t_ivs), 3)
        ph["intervals_only_output_bitwise_equal"] = bool(torch.equal(
            out_iv, csa.sparse_attn_fwd(q, k, v, plan, work, out=torch.empty_like(out))))
    ph["plan_bytes_intervals_only"] = plan_iv.nbytes()
    result["phases"] = ph
    # ---- e2e through the public API with host buffers (H2D of Q/K/V, D2H of O in the region)
    # csa.sparse_attn_fwd_host streams head chunks: H2D of chunk c+1 and D2H of chunk c-1
    # overlap the attention of chunk c (the same per-head arithmetic, bitwise)
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    ho = torch.empty(out.shape, dtype=out.dtype).pin_memory()

    def e2e_step():
        if B == 1:
            csa.sparse_attn_fwd_host(hq, hk, hv, plan, ho, heads_per_chunk=2, device=dev)
        else:  # batch > 1: whole-tensor copies around the device call
            dq, dk, dv = (t.to(dev, non_blocking=True) for t in (hq, hk, hv))
            ho.copy_(csa.sparse_attn_fwd(dq, dk, dv, plan, work, out=out), non_blocking=True)

    n_e2e = max(2, args.steps // 3)
    t_e2e, _, _ = time_loop(e2e_step, n_e2e, 1, stream)
    t_e2e /= n_e2e
    result["e2e"] = {"value": round(flop_all / (t_e2e * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                     "ms_per_step": round(t_e2e, 3),
                     "h2d_bytes_per_step": 3 * q.numel() * 2, "d2h_bytes_per_step": out.numel() * 2}
    result["gpu_launches"] = args.steps * launches_per_call(lay, cfg.d)


def reference_arm(args, cfg, world, rank):
    """--impl reference: the fp64 oracle, as it stands, on host cores.
    Each step = a bounded sample of (head, query-block) units of the same workload."""
    if rank != 0:
        return
    lay = cfg.layout
    world = world if "WORLD_SIZE" in os.environ else args.gpus
    # the same plan as our arm: generator S at the total sparsity, or (Mochi) the calibration
    # path, which needs the GPU
    _, masks, rep, _, _, _ = workload(cfg, args, 0, cfg.heads,
                                      torch.device("cuda" if cfg.sparsity is None else "cpu"))
    q, k, v = inputs.qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cpu")
    heads64 = OracleHeads(q, k, v)
    vals, t_steps = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb, _ = cpu_oracle_sample(lay, cfg, masks, rep, heads64, seconds_target=4.0)
        if i >= args.warmup:
            vals.append(cb["value"])
            t_steps.append(time.perf_counter() - t0)
    value = statistics.mean(vals)
    cb["value"] = round(value, 6)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(t_steps), 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(cfg, args.batch,
                             flops_of(lay, masks, rep, range(cfg.heads), cfg.d, 1)[1]
                             / (cfg.heads * float(lay.N) ** 2), rep, 1),
        "cpu_baseline": cb,
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
