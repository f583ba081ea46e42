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
    ap.add_argument("--workload", default="c3head", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--depth", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of a CUDA graph")
    ap.add_argument("--graph", action="store_true",
                    help="N > 1: capture the step (and its NCCL collectives) as a CUDA graph; the "
                         "default at N > 1 is eager launches (graph capture of the collectives has "
                         "not run on a multi-GPU box)")
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
    # TP_BENCH_DEVICE: every rank on that device (one-GPU multi-process test runs, tests/ncclshim)
    local = int(os.environ.get("TP_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        # torch.distributed is rendezvous + timing plumbing only (barriers, the max over ranks);
        # TP_BENCH_DIST_BACKEND=gloo is for one-GPU multi-process test runs (tests/ncclshim)
        backend = os.environ.get("TP_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        if not a.graph:
            a.eager = True

    def max_over_ranks(v):
        if world == 1:
            return v
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
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
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)  # L2 flush (not the model's)
    torch.cuda.synchronize()
    mem0 = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    model = TPMLP(g, M, layers, dtype=dtype, seed=a.seed,
                  flags=api.TP_FLAG_PEER_FUSED if fused else 0)
    x, ws_, dy_last, dacts, grads_w = model.x, model.W, model.dY, model.dX, model.dW
    step = model.step

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    barrier()
    mem_peak = torch.cuda.max_memory_allocated() - mem0
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
        prof_step_ms = 0.0
        for k in range(a.steps):
            api.tp_l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            gprof.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            prof_step_ms += e0.elapsed_time(e1)
            m_, n_, f_ = api.tp_prof_read(0)
            gemm_ms, gemm_n, gemm_flops = gemm_ms + m_, gemm_n + n_, gemm_flops + f_
            m_, n_, f_ = api.tp_prof_read(1)
            simt_ms, simt_n, simt_flops = simt_ms + m_, simt_n + n_, simt_flops + f_
        del gprof
    else:
        prof_step_ms = 0.0
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
    ms = max_over_ranks(sum(s.elapsed_time(e) for s, e in ev) / a.steps)
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
            return max_over_ranks(tot / n_e2e)

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

        # pipelined (the headline): a training loop's double buffering - step t+1's X and dY
        # copy in and step t's dX copies out on a copy stream while step t / t+1 compute; every
        # step still moves its own inputs and result across PCIe inside the timed region
        xb = [x, torch.empty_like(x)]
        dyb = [dy_last, torch.empty_like(dy_last)]
        dxb = [dacts[0], torch.empty_like(dacts[0])]
        hdxb = [hdx, torch.empty_like(hdx).pin_memory()]

        def pipelined_run(n):
            ev_in = [None] * n
            done = [None] * n
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                xb[0].copy_(hx, non_blocking=True)
                dyb[0].copy_(hdy, non_blocking=True)
                ev_in[0] = cs.record_event()
            for t in range(n):
                b = t % 2
                if t + 1 < n:
                    with torch.cuda.stream(cs):
                        if t >= 1:
                            cs.wait_event(done[t - 1])  # buffers 1-b free (step t-1 finished)
                        xb[1 - b].copy_(hx, non_blocking=True)
                        dyb[1 - b].copy_(hdy, non_blocking=True)
                        ev_in[t + 1] = cs.record_event()
                stream.wait_event(ev_in[t])
                model.x, model.dY, model.dX[0] = xb[b], dyb[b], dxb[b]
                model.forward()
                model.backward()
                done[t] = stream.record_event()
                with torch.cuda.stream(cs):
                    cs.wait_event(done[t])
                    hdxb[b].copy_(dxb[b], non_blocking=True)
            stream.wait_stream(cs)
            model.x, model.dY, model.dX[0] = x, dy_last, dacts[0]

        pipelined_run(2)  # warm-up
        barrier()
        api.tp_l2_flush(flush)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        pipelined_run(n_e2e)
        p1.record(stream)
        p1.synchronize()
        pms = max_over_ranks(p0.elapsed_time(p1) / n_e2e)
        ems = timed(resident)
        sms = timed(streamed)
        e2e = {"value": round(flops / (pms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(pms, 4), "h2d_bytes_per_step": nbytes([hx, hdy]),
               "d2h_bytes_per_step": nbytes([hdx]),
               "what": f"{n_e2e} consecutive steps timed as one region (total / steps): per step, "
                       "X and dY host->device and dX device->host (pinned host buffers, a copy "
                       "stream, device buffers double-buffered so step t+1's copies overlap step "
                       "t's compute), fwd+bwd through TPMLP / tp_linear_*; weights resident (W1, "
                       "W2 and dW1, dW2 stay in HBM for an on-device optimizer)",
               "unpipelined": {"value": round(flops / (ems * 1e-3) / 1e12, 3),
                               "ms_per_step": round(ems, 4),
                               "what": "each step timed alone: copies in, compute, copy out "
                                       "(dY's copy under the forward)"},
               "weights_streamed": {"value": round(flops / (sms * 1e-3) / 1e12, 3),
                                    "ms_per_step": round(sms, 4),
                                    "h2d_bytes_per_step": nbytes([hx, hdy] + hws),
                                    "d2h_bytes_per_step": nbytes(houts)}}

    pk, src = peaks()
    flops_gpu = flops / world                      # TP avoids no work: 6MKN/p per GPU per layer
    costs = [api.tp_cost_model(mode, world, d_, depth=depth) for d_ in model.descs]
    link_bytes = sum(c["link_bytes"] for c in costs)   # algorithmic NVLink bytes per GPU per step
    nvlink_gbs = 900.0                                 # NVLink 5 per direction per GPU
    if dtype == "bf16":
        # a short step times each GEMM alone (burst peak); a step of several ms keeps the GPU at
        # its power cap, where the sustained figure is the denominator (B200_PROFILING.md)
        long_step = ms > 5.0
        peak = pk.get("bf16_tflops_sustained" if long_step else "bf16_tflops")
        # achieved = the step's algorithmic GEMM flops per GPU / the uninstrumented timed step
        # (at p = 1 every flop of the step is a GEMM flop; collectives count as step time)
        ach = flops_gpu / (ms * 1e-3) / 1e12
        kern = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        roof = {"bound": "tensor", "kernel": "gemm_tc2_kernel / gemm_tc_kernel (tcgen05, bf16->fp32)",
                "achieved": round(ach, 2), "peak": peak, "unit": "TFLOP/s",
                "frac": round(ach / peak, 4),
                "achieved_from": "step GEMM flops per GPU / ms_per_step (uninstrumented timed step)",
                "peak_source": src + (" bf16_tflops_sustained (long step)" if long_step
                                      else " bf16_tflops (burst)"),
                "traffic": traffic_of(a.workload, world), "traffic_unit": "bytes/launch (ncu)",
                "alg_bytes_per_gemm": alg_bytes_per_gemm(M, layers, world, mode),
                "alg_bytes_per_step": (sum(2 * (M * K + K * N + M * N) * 3 for K, N in layers)
                                       if world == 1 else None),
                "breakdown": {
                    "gemm_launches_per_step": gemm_n // max(a.steps, 1),
                    "gemm_kernel_tflops": round(kern, 2) if kern else None,
                    "gemm_share_of_step": (round(min(1.0, gemm_ms / prof_step_ms), 3)
                                           if prof_step_ms > 0 else None),
                    "how": "per-GEMM CUDA events on the launching stream (external event nodes "
                           "in a separately captured graph), share = their sum / the same "
                           "instrumented replays' step time"}}
        # which roof binds: flops at the tensor peak vs algorithmic operand + output bytes at the
        # measured HBM bandwidth (p = 1; e.g. C3's 64-row GEMMs stream a 512 MB weight each)
        step_b = roof["alg_bytes_per_step"]
        hbm = pk.get("hbm_gbs")
        t_tensor = flops_gpu / (peak * 1e12)
        if step_b and hbm:
            t_hbm = step_b / (hbm * 1e9)
            if t_hbm > t_tensor:
                gbs = step_b / (ms * 1e-3) / 1e9
                roof.update({"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(gbs / hbm, 4), "peak_source": src + " hbm_gbs",
                             "tensor_achieved_tflops": round(ach, 2),
                             "tensor_frac": round(ach / peak, 4)})
            roof["roof_times_us_per_step"] = {"tensor": round(t_tensor * 1e6, 1),
                                              "hbm": round(t_hbm * 1e6, 1)}
        if world > 1:
            # the second roof of a sharded step: the schedule's algorithmic NVLink bytes per GPU
            # (tp_cost_model) at 900 GB/s per direction
            t_link = link_bytes / (nvlink_gbs * 1e9)
            roof["nvlink"] = {"bytes_per_gpu_per_step": link_bytes,
                              "achieved_gbs": round(link_bytes / (ms * 1e-3) / 1e9, 1),
                              "peak_gbs": nvlink_gbs, "frac": round(link_bytes / (ms * 1e-3) / 1e9
                                                                    / nvlink_gbs, 4)}
            roof["roof_times_us_per_step"] = {"tensor": round(t_tensor * 1e6, 1),
                                              "nvlink": round(t_link * 1e6, 1)}
            if t_link > t_tensor:
                roof["bound"] = "nvlink"
            roof["frac_of_roofline"] = round(max(t_tensor, t_link) / (ms * 1e-3), 4)
    else:
        peak = 148 * 128 * 2 * 1.965  # fp32 FFMA: SMs x lanes x 2 flop x GHz (GFLOP/s->TFLOP/s /1e3)
        peak = peak / 1e3
        ach = flops_gpu / (ms * 1e-3) / 1e12
        roof = {"bound": "alu", "kernel": "gemm_simt_kernel (fp32 FFMA)", "achieved": round(ach, 4),
                "peak": round(peak, 2), "unit": "TFLOP/s", "frac": round(ach / peak, 5),
                "traffic": None}

    # per-rank device memory: the paper's measurement ("max allocated CUDA memory")
    # next to its closed form (at-rest shards of X, Y1, Y2, W1, W2 from tp_cost_model) and the
    # closed form of everything the step allocates (+ dY, dX_i, dW_i, workspace, saved)
    esz = 2 if dtype == "bf16" else 4
    at_rest = (costs[0]["mem_x"] + sum(c["mem_w"] + c["mem_y"] for c in costs)) * esz
    nb = lambda t: t.numel() * t.element_size() if t is not None else 0
    allocated = (nb(model.x) + sum(map(nb, model.W)) + sum(map(nb, model.Y)) + nb(model.dY)
                 + sum(map(nb, model.dX)) + sum(map(nb, model.dW)) + nb(model.ws)
                 + sum(map(nb, model.saved)))
    mem = {"peak_allocated_bytes": int(mem_peak),
           "closed_form_at_rest_bytes": int(at_rest),
           "closed_form_step_bytes": int(allocated),
           "peak_over_step_closed_form": round(mem_peak / allocated, 4) if allocated else None,
           "how": "torch.cuda.max_memory_allocated over model build + warm-up steps, minus the "
                  "allocation before the model; closed forms: tp_cost_model shard sizes"}

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
        "memory_per_rank": mem,
        # library tuning knobs not at their measured defaults (tp_knobs): empty in a normal run
        "tuning_overrides": {k["name"]: k["value"] for k in api.tp_knobs() if k["source"] != "default"},
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

def oracle_setup(wl, mode, world, depth, seed, max_rows):
    """The oracle's inputs, generated ONCE outside every timed region: the first `max_rows` rows
    of the global X and dY (a row sample of the batch) and the full weights, in fp64. Returns a
    closure building the rank-by-rank shards for a sample of M rows (also untimed)."""
    import numpy as np
    import synth
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec, shard
    layers, dt = wl["layers"], wl["dtype"]
    g = build_grid(mode, world, depth)
    X = synth.tensor(seed, 0, wl["M"], layers[0][0], dtype=dt, nrows=max_rows).astype(np.float64)
    Ws = [synth.tensor(seed, 16 * i + 1, K, N, scale=synth.xavier_scale(K, N), dtype=dt)
          .astype(np.float64) for i, (K, N) in enumerate(layers)]
    dY = synth.tensor(seed, 16 * (len(layers) - 1) + 2, wl["M"], layers[-1][1], dtype=dt,
                      nrows=max_rows).astype(np.float64)

    def for_rows(M):
        specs = [LayerSpec(M, K, N, split_1d="row" if i % 2 else "col", parity=i % 2)
                 for i, (K, N) in enumerate(layers)]
        return {"g": g, "specs": specs, "X": shard(g, specs[0], X[:M], "X"),
                "W": [shard(g, sp, W, "W") for sp, W in zip(specs, Ws)],
                "dY": shard(g, specs[-1], dY[:M], "Y"),
                "flops": sum(6.0 * M * K * N for K, N in layers)}
    return for_rows


def oracle_step(st):
    """One fwd+bwd of the layer chain through the oracle's rank-by-rank programs (the timed
    work: the per-rank GEMMs and simulated collectives only). Returns the sample's flops."""
    from oracle import programs
    from oracle.fabric import Fabric
    g, specs, fab = st["g"], st["specs"], Fabric()
    acts, saves = [st["X"]], []
    for i, sp in enumerate(specs):
        Y, sv = programs.layer_fwd(g, sp, acts[-1], st["W"][i], fab=fab)
        acts.append(Y)
        saves.append(sv)
    dy = st["dY"]
    for i in reversed(range(len(specs))):
        dy, _, _ = programs.layer_bwd(g, specs[i], dy, acts[i], st["W"][i], fab=fab, saved=saves[i])
    return st["flops"]


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), None)
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": model}


def one_blas_thread():
    """The oracle is timed single-threaded: BLAS pinned to one thread."""
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=1, user_api="blas")


def oracle_sample(a, mode, world, depth, step_s):
    """Inputs generated once; the row sample sized (by a calibration step) so that one oracle
    step takes about step_s seconds on one core. Returns (state, M_run, M_full)."""
    wl = WORKLOADS[a.workload]
    M_full = wl["M"]
    unit, gd = 1, grid_dims(mode, world, depth)
    if mode == "2d":
        unit = gd[0]
    elif mode == "2.5d":
        unit = gd[0] * gd[1]
    elif mode == "3d":
        unit = gd[0] * gd[0]
    unit = max(unit, 8)
    cap = min(M_full, 64 * unit)
    build = oracle_setup(wl, mode, world, depth, a.seed, cap)
    M_cal = min(M_full, unit)
    with one_blas_thread():
        st = build(M_cal)
        t0 = time.perf_counter()
        oracle_step(st)
        rate = st["flops"] / (time.perf_counter() - t0)
    per_row = st["flops"] / M_cal
    M_run = int(step_s * rate / per_row) // unit * unit
    M_run = max(unit, min(cap, M_run))
    return build(M_run), M_run, M_full


def cpu_baseline(a, mode, world, depth, budget_s=15.0):
    st, M_run, M_full = oracle_sample(a, mode, world, depth, budget_s / 3)
    n, fl = 0, 0.0
    with one_blas_thread():
        t0 = time.perf_counter()
        while n < 3 and (n == 0 or time.perf_counter() - t0 < budget_s):
            fl += oracle_step(st)
            n += 1
        dt = time.perf_counter() - t0
    return {"value": round(fl / dt / 1e12, 6), "unit": "TFLOP/s", "cores": 1, **host_info(),
            "kind": "oracle",
            "sample": f"{n} oracle step(s) of {a.workload} {mode} p={world}, rows 0..{M_run} of "
                      f"{M_full} (full weights); fp64 numpy rank-by-rank program, BLAS on 1 thread, "
                      f"inputs generated before timing; {dt:.1f} s"}


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[a.workload]
    mode = DEFAULT_MODE.get(world, "1d") if a.mode == "auto" else a.mode
    depth = a.depth if mode == "2.5d" else 1
    # each step: a bounded row sample of the workload (~1 s of one core), inputs generated once
    st, M_run, M = oracle_sample(a, mode, world, depth, 1.0)
    with one_blas_thread():
        for _ in range(a.warmup):
            oracle_step(st)
        t0 = time.perf_counter()
        fl = 0.0
        for _ in range(a.steps):
            fl += oracle_step(st)
        dt = time.perf_counter() - t0
    v = fl / dt / 1e12
    line = {"impl": "reference", "metric": METRIC,
            "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(dt / a.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(a.workload, mode, depth, world),
            "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "kind": "oracle", "cores": 1,
                             **host_info(),
                             "sample": f"rows 0..{M_run} of {M} per step (full weights), fp64 "
                                       f"numpy rank-by-rank oracle, BLAS on 1 thread, inputs "
                                       f"generated before timing"},
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
