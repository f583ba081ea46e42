"""Benchmark of the tensor-parallel linear layer (fwd + bwd of two linear layers).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--mode auto]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...     # the fp64 CPU oracle, same metric (rank 0 only)

One step = the whole hot path over one batch: Y1 = X.W1 (layer 1), Y2 = Y1.W2 (layer 2),
then backward of layer 2 (dY1, dW2) and layer 1 (dX, dW1), all through the C ABI
(include/tp_b200.h). Inputs are seeded synthetic tensors generated on device by the
library's generator (same recipe as synth/), resident in HBM before timing; L2 is flushed
(256 MiB write) between timed steps, outside the timed events.

Prints ONE JSON line (rank 0). value = whole-job TFLOP/s (sum over GPUs of 6*M*K*N per
layer / max-over-ranks device time).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# one metric string for both arms (BASELINE.json metric; value = whole-job TFLOP/s)
METRIC = "TP linear fwd+bwd TFLOP/s (whole job; per-GPU in per_gpu_tflops) + % of roofline"

# BASELINE.json configs -> (M tokens, hidden, layer widths)
WORKLOADS = {
    "c1": dict(M=16, layers=[(64, 64), (64, 64)], dtype="fp32",
               desc="configs[0]: two linear layers, batch 16 x hidden 64, fp32"),
    "c2": dict(M=512, layers=[(4096, 4096), (4096, 4096)], dtype="bf16",
               desc="configs[1]: paper range test, two linear layers, batch 512, hidden 4096, bf16"),
    "c3": dict(M=64, layers=[(16384, 16384), (16384, 16384)], dtype="bf16",
               desc="configs[2]: range test by hidden, batch 64, hidden 16384, bf16"),
    "c3head": dict(M=16384, layers=[(16384, 16384), (16384, 16384)], dtype="bf16",
                   desc="configs[2] HEAD reading: 64 x 256 = 16384 tokens, hidden 16384, bf16"),
    "c4": dict(M=4096 * 197, layers=[(384, 1536), (1536, 384)], dtype="bf16",
               desc="configs[3]: ViT-S/16 MLP (fc1 384->1536, fc2 1536->384), 197 tokens x batch 4096"),
    "c5": dict(M=16384, layers=[(8192, 32768), (32768, 8192)], dtype="bf16",
               desc="configs[4]: GPT MLP h=8192, seq 2048 x batch 8, bf16"),
}

DEFAULT_MODE = {1: "1d", 2: "1d", 4: "2d", 8: "3d"}


def grid_dims(mode, world, depth):
    if mode == "1d":
        return [world]
    if mode == "2d":
        q = round(world ** 0.5)
        return [q, q]
    if mode == "2.5d":
        q = round((world // depth) ** 0.5)
        return [depth, q, q]
    l = round(world ** (1 / 3))
    return [l, l, l]


def config_of(workload, mode, depth, world, fused=False):
    """The bench line's `config` (identical on both arms)."""
    wl = WORKLOADS[workload]
    M, layers = wl["M"], wl["layers"]
    return {"workload": workload, "desc": wl["desc"], "mode": mode, "depth": depth,
            "grid": grid_dims(mode, world, depth), "M": M, "layers": layers,
            "flops_per_step": float(sum(6.0 * M * K * N for K, N in layers)),
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": f"tp-{mode}x{world}" + ("-fused" if fused else "")}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--fused", action="store_true",
                    help="N > 1: fused peer-panel schedule (TP_FLAG_PEER_FUSED; 2D / 2.5D / 3D l=2)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        mx = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def traffic_of(workload, world):
    """DRAM bytes (read + write) per GEMM launch from the committed ncu capture of this workload
    (tools/ncu_traffic.py writes profiles/traffic_<workload>_p<N>.json), else None."""
    p = os.path.join(ROOT, "profiles", f"traffic_{workload}_p{world}.json")
    try:
        with open(p) as f:
            return json.load(f)["dram_bytes_per_gemm_launch"]
    except (OSError, KeyError, ValueError):
        return None


def alg_bytes_per_gemm(M, layers, world, mode):
    """Algorithmic HBM bytes per GEMM launch at p = 1: each operand read once, output written
    once (bf16), averaged over the step's 3 GEMMs per layer (fwd, dX, dW)."""
    if world != 1:
        return None
    tot = 0
    for K, N in layers:
        tot += 2 * (M * K + K * N + M * N) * 3
    return tot // (3 * len(layers))


# ------------------------------------------------------------------------------- our arm

def layer_descs(api, mode, M, layers, dtype):
    ds = []
    for li, (K, N) in enumerate(layers):
        ds.append(api.desc(M, K, N, dtype, split_1d=li % 2, parity_3d=li % 2))
    return ds


def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2110_14883_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[a.workload]
    mode = DEFAULT_MODE.get(world, "1d") if a.mode == "auto" else a.mode
    depth = a.depth if mode == "2.5d" else 1
    M, layers, dtype = wl["M"], wl["layers"], wl["dtype"]
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32

    if world > 1:
        uid = api.share_unique_id(api.TP_TRANSPORT_NCCL)
        g = api.tp_grid_init(mode, world, rank, 0, depth, local, api.TP_TRANSPORT_NCCL, uid)
    else:
        g = api.tp_grid_init(mode, 1, 0, 0, 1, local, api.TP_TRANSPORT_NONE)
    # ---- this rank's shards, generated in place by the library's seeded generator ----
    from paper_2110_14883_b200.mlp import TPMLP
    fused = a.fused and world > 1
    model = TPMLP(g, M, layers, dtype=dtype, seed=a.seed,
                  flags=api.TP_FLAG_PEER_FUSED if fused else 0)
    x, ws_, dy_last, dacts, grads_w = model.x, model.W, model.dY, model.dX, model.dW
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    step = model.step

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    barrier()
    stream = torch.cuda.current_stream()

    # ---- pass 1 (instrumented): CUDA events around every GEMM launch on its launching stream
    # (captured into the step's graph as external event nodes) -> the dominant kernel's
    # achieved TFLOP/s for the roofline; kernel launches per step
    api.tp_prof_reset()
    n0 = api.tp_launch_count()
    api.tp_prof_enable(True)
    gemm_ms = gemm_flops = simt_ms = simt_flops = 0.0
    gemm_n = simt_n = 0
    if not a.eager:
        gprof = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gprof):
            step()
        api.tp_prof_enable(False)
        launches_per_step = api.tp_launch_count() - n0
        for k in range(a.steps):
            api.tp_l2_flush(flush)
            gprof.replay()
            torch.cuda.synchronize()
            m_, n_, f_ = api.tp_prof_read(0)
            gemm_ms, gemm_n, gemm_flops = gemm_ms + m_, gemm_n + n_, gemm_flops + f_
            m_, n_, f_ = api.tp_prof_read(1)
            simt_ms, simt_n, simt_flops = simt_ms + m_, simt_n + n_, simt_flops + f_
        del gprof
    else:
        for k in range(a.steps):
            api.tp_l2_flush(flush)
            torch.cuda._sleep(2_000_000)   # host runs ahead: events bracket device time only
            step()
            torch.cuda.synchronize()
        api.tp_prof_enable(False)
        launches_per_step = (api.tp_launch_count() - n0) // a.steps
        gemm_ms, gemm_n, gemm_flops = api.tp_prof_read(0)
        simt_ms, simt_n, simt_flops = api.tp_prof_read(1)
    barrier()
    api.tp_prof_reset()

    # ---- pass 2 (timed): the step captured once as a CUDA graph (all of its kernels and
    # collectives, no host work per step), replayed K times, L2 flushed between replays
    graph = None
    if not a.eager:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(a.warmup):
            graph.replay()
        barrier()
    run_step = graph.replay if graph is not None else step
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    with Clocks(local) as clk:
        t_wall = time.perf_counter()
        for k in range(a.steps):
            api.tp_l2_flush(flush)
            ev[k][0].record(stream)
            run_step()
            ev[k][1].record(stream)
        barrier()
        t_wall = time.perf_counter() - t_wall
    launches = launches_per_step * a.steps
    ms = sum(s.elapsed_time(e) for s, e in ev) / a.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = sum(6.0 * M * K * N for K, N in layers)
    value = flops / (ms * 1e-3) / 1e12

    # ---- end to end through the public API (TPMLP.forward / backward -> tp_linear_fwd/bwd):
    # host buffers, copies inside the timed region. Per step the host supplies the step's
    # inputs X and dY (pinned) and reads back its result dX; the weights are the model's
    # resident state (as in training: W stays in HBM, dW feeds an on-device optimizer). dY's
    # copy runs on a side stream under the forward. For transparency the run also measures
    # the weights-streamed variant (every W in, every dW out, serial on one stream).
    e2e = None
    if not a.no_e2e:
        hx = x.cpu().pin_memory()
        hws = [w.cpu().pin_memory() for w in ws_]
        hdy = dy_last.cpu().pin_memory()
        hdx = torch.empty(dacts[0].shape, dtype=dacts[0].dtype).pin_memory()
        outs = [dacts[0]] + grads_w
        houts = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
        nbytes = lambda ts: sum(t.numel() * t.element_size() for t in ts)
        cs = torch.cuda.Stream()
        n_e2e = max(3, a.steps // 2)

        def timed(one):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tot = 0.0
            for _ in range(n_e2e):
                api.tp_l2_flush(flush)
                e0.record(stream)
                one()
                e1.record(stream)
                e1.synchronize()
                tot += e0.elapsed_time(e1)
            t_ms = tot / n_e2e
            if world > 1:
                t = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                t_ms = float(t.item())
            return t_ms

        def resident():
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                dy_last.copy_(hdy, non_blocking=True)
            x.copy_(hx, non_blocking=True)
            model.forward()
            stream.wait_stream(cs)
            model.backward()
            hdx.copy_(dacts[0], non_blocking=True)

        def streamed():
            x.copy_(hx, non_blocking=True)
            for w, hw in zip(ws_, hws):
                w.copy_(hw, non_blocking=True)
            dy_last.copy_(hdy, non_blocking=True)
            step()
            for o, ho in zip(outs, houts):
                ho.copy_(o, non_blocking=True)

        ems = timed(resident)
        sms = timed(streamed)
        e2e = {"value": round(flops / (ems * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(ems, 4), "h2d_bytes_per_step": nbytes([hx, hdy]),
               "d2h_bytes_per_step": nbytes([hdx]),
               "what": "per step: X and dY host->device (dY on a side stream under the forward), "
                       "fwd+bwd through TPMLP / tp_linear_*, dX device->host; weights resident",
               "weights_streamed": {"value": round(flops / (sms * 1e-3) / 1e12, 3),
                                    "ms_per_step": round(sms, 4),
                                    "h2d_bytes_per_step": nbytes([hx, hdy] + hws),
                                    "d2h_bytes_per_step": nbytes(houts)}}

    pk, src = peaks()
    if dtype == "bf16":
        # a short step times each GEMM alone (burst peak); a step of several ms keeps the GPU at
        # its power cap, where the sustained figure is the denominator (B200_PROFILING.md)
        long_step = ms > 5.0
        peak = pk.get("bf16_tflops_sustained" if long_step else "bf16_tflops")
        ach = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        roof = {"bound": "tensor", "kernel": "gemm_tc_kernel / gemm_tc2_kernel (tcgen05, bf16->fp32)",
                "achieved": round(ach, 2) if ach else None, "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4) if ach else None,
                "peak_source": src + (" bf16_tflops_sustained (long step)" if long_step
                                      else " bf16_tflops (burst)"),
                "traffic": traffic_of(a.workload, world), "traffic_unit": "bytes/launch (ncu)",
                "alg_bytes_per_gemm": alg_bytes_per_gemm(M, layers, world, mode),
                "alg_bytes_per_step": (sum(2 * (M * K + K * N + M * N) * 3 for K, N in layers)
                                       if world == 1 else None),
                "launches_timed": gemm_n,
                "gemm_share_of_step": round(gemm_ms / a.steps / ms, 3) if ms > 0 else None,
                "timing": "per-GEMM CUDA events on the launching stream, recorded inside the "
                          "step graph (external event nodes), K instrumented replays"}
        # which roof binds the GEMM family: algorithmic flops at the tensor peak vs algorithmic
        # operand + output bytes at the measured HBM bandwidth (p = 1; e.g. C3's 64-row GEMMs
        # stream a 512 MB weight per launch and are HBM-bound)
        step_b = roof["alg_bytes_per_step"]
        hbm = pk.get("hbm_gbs")
        if ach and step_b and hbm and gemm_n:
            t_tensor = gemm_flops / (peak * 1e12)
            t_hbm = step_b * a.steps / (hbm * 1e9)
            if t_hbm > t_tensor:
                gbs = step_b * a.steps / (gemm_ms * 1e-3) / 1e9
                roof.update({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(gbs / hbm, 4), "peak_source": src + " hbm_gbs",
                             "tensor_achieved_tflops": round(ach, 2),
                             "tensor_frac": round(ach / peak, 4)})
            roof["roof_times_us_per_step"] = {"tensor": round(t_tensor / a.steps * 1e6, 1),
                                              "hbm": round(t_hbm / a.steps * 1e6, 1)}
    else:
        peak = 148 * 128 * 2 * 1.965  # fp32 FFMA: SMs x lanes x 2 flop x GHz (GFLOP/s->TFLOP/s /1e3)
        peak = peak / 1e3
        ach = simt_flops / (simt_ms * 1e-3) / 1e12 if simt_ms > 0 else None
        roof = {"bound": "alu", "kernel": "gemm_simt_kernel (fp32 FFMA)", "achieved": ach,
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": (ach / peak) if ach else None,
                "traffic": None}

    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a, mode, world, depth)

    line = {
        "metric": METRIC,
        "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if dtype == "bf16" else "f32",
        "data": "synthetic (seeded SplitMix64, Xavier-uniform W, U(-1,1) X/dY; generated in HBM)",
        "config": config_of(a.workload, mode, depth, world, fused),
        "per_gpu_tflops": round(value / world, 3),
        "wall_s": round(t_wall, 3),
        "launch": "cuda-graph replay" if graph is not None else "eager",
        "gpu_launches": launches,
        "roofline": roof,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    api.tp_grid_destroy(g)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------- oracle arm

def oracle_step(wl, mode, world, depth, seed, M_sample=None):
    """One fwd+bwd of the two-layer model through the oracle's rank-by-rank programs.
    Returns flops of the sample."""
    import numpy as np
    import synth
    from oracle import programs
    from oracle.fabric import Fabric
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec, shard
    M = wl["M"] if M_sample is None else M_sample
    layers = wl["layers"]
    g = build_grid(mode, world, depth)
    specs = [LayerSpec(M, K, N, split_1d="row" if i % 2 else "col", parity=i % 2)
             for i, (K, N) in enumerate(layers)]
    fab = Fabric()
    X = synth.tensor(seed, 0, M, layers[0][0], dtype=wl["dtype"]).astype(np.float64)
    acts = [shard(g, specs[0], X, "X")]
    Ws, saves = [], []
    for i, (K, N) in enumerate(layers):
        W = synth.tensor(seed, 16 * i + 1, K, N, scale=synth.xavier_scale(K, N), dtype=wl["dtype"])
        Ws.append(shard(g, specs[i], W.astype(np.float64), "W"))
        Y, sv = programs.layer_fwd(g, specs[i], acts[-1], Ws[-1], fab=fab)
        acts.append(Y)
        saves.append(sv)
    dY = synth.tensor(seed, 16 * (len(layers) - 1) + 2, M, layers[-1][1], dtype=wl["dtype"])
    dy = shard(g, specs[-1], dY.astype(np.float64), "Y")
    for i in reversed(range(len(layers))):
        dy, _, _ = programs.layer_bwd(g, specs[i], dy, acts[i], Ws[i], fab=fab, saved=saves[i])
    return sum(6.0 * M * K * N for K, N in layers)


def oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def cpu_baseline(a, mode, world, depth, budget_s=12.0):
    wl = WORKLOADS[a.workload]
    M_s = wl["M"]
    # bounded sample: shrink the batch (rows) until one oracle step fits the budget
    t0 = time.perf_counter()
    fl = oracle_step(wl, mode, world, depth, a.seed, min(M_s, 64 * world * world))
    dt = time.perf_counter() - t0
    rate = fl / dt
    full = sum(6.0 * M_s * K * N for K, N in wl["layers"])
    M_run = M_s if full / rate <= budget_s else max(world * world, int(M_s * budget_s * rate / full))
    M_run = max(world * world * depth, (M_run // (world * world * depth)) * world * world * depth)
    t0 = time.perf_counter()
    n, fl_tot = 0, 0.0
    while True:
        fl_tot += oracle_step(wl, mode, world, depth, a.seed, M_run)
        n += 1
        if time.perf_counter() - t0 > 0.5 * budget_s or n >= 3:
            break
    dt = time.perf_counter() - t0
    return {"value": round(fl_tot / dt / 1e12, 6), "unit": "TFLOP/s", "cores": oracle_threads(),
            "kind": "oracle",
            "sample": f"{n} oracle step(s) of {a.workload} {mode} p={world} with M={M_run} rows "
                      f"(of {M_s}); fp64 numpy rank-by-rank program, {dt:.1f} s"}


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[a.workload]
    mode = DEFAULT_MODE.get(world, "1d") if a.mode == "auto" else a.mode
    depth = a.depth if mode == "2.5d" else 1
    M = wl["M"]
    unit = world * world * depth
    # each step: a bounded sample of the workload (rows) sized so the run stays ~minutes
    M_run = max(unit, min(M, 128 * unit) // unit * unit)
    for _ in range(a.warmup):
        oracle_step(wl, mode, world, depth, a.seed, M_run)
    t0 = time.perf_counter()
    fl = 0.0
    for _ in range(a.steps):
        fl += oracle_step(wl, mode, world, depth, a.seed, M_run)
    dt = time.perf_counter() - t0
    v = fl / dt / 1e12
    line = {"impl": "reference", "metric": METRIC,
            "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(dt / a.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(a.workload, mode, depth, world),
            "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "kind": "oracle",
                             "cores": oracle_threads(),
                             "sample": f"M={M_run} of {M} rows per step, fp64 numpy oracle"},
            "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.warmup < 3:
        a.warmup = 3
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
