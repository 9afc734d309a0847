"""Benchmark of the complex-Winograd int8 3x3 conv hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = the whole hot path over one batch of
synthetic input: filter transform + scaling (K1) and the convolution
(K2 input transform -> K3F fused tcgen05 GEMMs + reverse scaling + output
transform, per chunk; `--path staged` runs the three-kernel K2 -> K3 -> K4 path).
Weak scaling: every rank runs its own batch of the configuration (data
parallel by batch, no collective on the data path).  Inputs and weights are
rotated over enough distinct sets that they never stay resident in the 126 MB
L2 between steps.  Rank 0 prints one JSON line.

`--impl reference` times the CPU oracle (oracle/, plain C) on the host cores,
one bounded sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "int8 3x3 conv effective TOPS (direct-conv ops/s)"
L2_BYTES = 126 * 2 ** 20


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def _peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    return {
        "hbm_gbs": float(p.get("hbm_gbs", 6650.0)),
        "bf16_tflops": float(p.get("bf16_tflops", 1590.0)),
        "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", 1400.0)),
        "source": "MEASURED_PEAKS.json (measured)" if p else "B200_PROFILING.md fallback",
    }


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while running."""

    def __init__(self, dev_index: int, period_s: float = 0.01):
        self.dev_index, self.period = dev_index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self.nv = None
            self.err = str(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1901_01965_b200 as W
    from paper_1901_01965_b200 import _lib as L

    rank, local_rank, world = _env_rank()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    from paper_1901_01965_b200 import shard as SH
    cfg = synth.CONFIGS[args.config]
    layer = cfg.layers[0]
    S = synth.requant_shift(layer)
    # weak: every rank runs the whole configuration on its own batch; strong: the
    # configuration's batch (or Cout for batch < world) is split over the ranks
    sh = SH.shard(layer.n, layer.c_out, world, rank) if args.scaling == "strong" else \
        {"mode": "replica", "n0": 0, "n": layer.n, "co0": 0, "co": layer.c_out}
    path = {"staged": W.WINO_PATH_STAGED, "fused": W.WINO_PATH_FUSED, "auto": W.WINO_PATH_AUTO}[args.path]
    alg = W.WINO_ALG_F2X2 if args.alg == "f2" else W.WINO_ALG_F4X4
    # --input u8: the same synthetic values as uint8 tensors with zero points 128
    u8 = args.input == "u8"
    zp = 128 if u8 else 0
    conv = W.WinoConv2d(sh["n"], layer.h, layer.w, layer.c_in, sh["co"], layer.pad, W.WINO_NHWC, layer.scaling,
                        W.WINO_OUT_INT8, device=local_rank, path=path, algorithm=alg,
                        input_type=W.WINO_IN_UINT8 if u8 else W.WINO_IN_INT8, x_zero_point=zp, w_zero_point=zp,
                        filter_target_max=args.target)
    to_in = (lambda a: (a.astype(np.int16) + 128).astype(np.uint8)) if u8 else (lambda a: a)
    info = conv.info
    x_bytes, y_bytes = info.x_bytes, info.y_bytes
    w_bytes = sh["co"] * 9 * layer.c_in
    per_set = x_bytes + w_bytes + y_bytes
    n_sets = max(2, math.ceil(1.2 * L2_BYTES / per_set))
    xs, ws, ys = [], [], []
    for i in range(n_sets):
        # first set: the seeded config tensors; later sets: re-seeded batches of the same recipe
        if args.scaling == "strong":   # global tensors, this rank's slice
            x, w = synth.config_inputs(args.config, rank=i)
            x = x[sh["n0"]: sh["n0"] + sh["n"]]
            w = np.ascontiguousarray(w[sh["co0"]: sh["co0"] + sh["co"]])
        else:
            x, w = synth.config_inputs(args.config, rank=rank * 1000 + i)
        xs.append(torch.from_numpy(np.ascontiguousarray(to_in(x))).to(dev))
        ws.append(torch.from_numpy(np.ascontiguousarray(to_in(w))).to(dev))
        ys.append(torch.empty(conv.y_shape, dtype=torch.int8, device=dev))
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    w_wino, codes, wsp = conv.w_wino.data_ptr(), conv.codes.data_ptr(), conv.workspace.data_ptr()
    # --streams > 1: independent batches in flight on separate streams, each with its own
    # transformed-filter buffer, codes and workspace (no dependencies between them)
    lanes = [(stream, conv.w_wino, conv.codes, conv.workspace)]
    for _ in range(1, max(1, args.streams)):
        lanes.append((torch.cuda.Stream(device=dev), torch.empty_like(conv.w_wino), torch.empty_like(conv.codes),
                      torch.empty_like(conv.workspace)))

    # --overlap-filter: the filter transform (K1) runs on a side stream concurrently with the
    # input transform (K2) of the same step; the GEMM waits for both (same work, fork/join inside
    # the captured graph).  Otherwise K1 -> conv on one stream.
    sides = [torch.cuda.Stream(device=dev) for _ in lanes]

    def step(i, lane=0):
        j = i % n_sets
        st_, ww_, cd_, ws_ = lanes[lane]
        if not args.overlap_filter:
            L.wino_transform_filter(conv.plan, ws[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), st_.cuda_stream)
            L.wino_conv2d_int8(conv.plan, xs[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), 1, S, ys[j].data_ptr(),
                               ws_.data_ptr(), st_.cuda_stream)
            return
        side = sides[lane]
        e_fork, e_join = torch.cuda.Event(), torch.cuda.Event()
        e_fork.record(st_)
        side.wait_event(e_fork)
        L.wino_transform_filter(conv.plan, ws[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), side.cuda_stream)
        e_join.record(side)
        for c in range(info.n_chunks):
            L.wino_conv2d_int8_stage(conv.plan, 2, c, xs[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), 1, S,
                                     ys[j].data_ptr(), ws_.data_ptr(), st_.cuda_stream)
            if c == 0:
                st_.wait_event(e_join)
            for stg in range(3, 2 + info.stages):
                L.wino_conv2d_int8_stage(conv.plan, stg, c, xs[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), 1,
                                         S, ys[j].data_ptr(), ws_.data_ptr(), st_.cuda_stream)

    launches_per_step = 1 + info.stages * info.n_chunks
    # CUDA graphs: one per (stream lane, rotation slot) (launch-bound otherwise)
    graphs = {}
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
        stream.synchronize()
        if not args.no_graph:
            for ln, (st_, _, _, _) in enumerate(lanes):
                with torch.cuda.stream(st_):
                    for j in range(n_sets):
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=st_):
                            step(j, ln)
                        graphs[(ln, j)] = g
                    for j in range(max(args.warmup, 3)):
                        graphs[(ln, j % n_sets)].replay()
            torch.cuda.synchronize()

    def run_steps(k, offset=0):
        n_l = len(lanes)
        for i in range(k):
            ln = i % n_l
            st_ = lanes[ln][0]
            with torch.cuda.stream(st_):
                if graphs:
                    graphs[(ln, (i + offset) % n_sets)].replay()
                else:
                    step(i + offset, ln)

    # ---------------- timed region
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for st_, _, _, _ in lanes[1:]:
            st_.wait_event(ev0)
        run_steps(args.steps)
        for st_, _, _, _ in lanes[1:]:
            e_ = torch.cuda.Event()
            e_.record(st_)
            stream.wait_event(e_)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_local = ev0.elapsed_time(ev1) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    ops_step = synth.direct_ops(layer)                     # one rank's configuration
    job_ops = ops_step * (world if args.scaling == "weak" else 1)
    value = job_ops * args.steps / t_max / 1e12

    # ---------------- per-kernel durations (roofline), same stream, outside the timed region
    kern = profile_kernels(conv, xs, ws, ys, S, stream, n_sets, 60)
    # ---------------- strong scaling: gather the sharded outputs of set 0 over NCCL (checking only,
    # outside the timed region) and compare them with rank 0's single-GPU run of the whole problem
    sharded_check = None
    if world > 1 and args.scaling == "strong":
        y_loc = conv(xs[0], 1, S)
        full_shape = (layer.n, conv.y_shape[1], conv.y_shape[2], layer.c_out)
        y_all = SH.gather_nhwc(y_loc, full_shape, sh, world, dev)
        if rank == 0:
            xf, wf = synth.config_inputs(args.config, rank=0)
            cf = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, layer.pad, W.WINO_NHWC,
                              layer.scaling, W.WINO_OUT_INT8, device=local_rank, path=path, algorithm=alg,
                              input_type=conv.desc.input_type, x_zero_point=zp, w_zero_point=zp,
                              filter_target_max=args.target)
            cf.transform_filter(torch.from_numpy(np.ascontiguousarray(to_in(wf))).to(dev))
            y_one = cf(torch.from_numpy(np.ascontiguousarray(to_in(xf))).to(dev), 1, S)
            sharded_check = {"mode": sh["mode"], "gathered_bytes": int(y_all.numel()),
                             "collective": "all_gather_into_tensor (NCCL), checking only",
                             "equal_to_single_gpu": bool(torch.equal(y_all, y_one))}
    # ---------------- scaling-induced error against direct convolution (outside the timed region)
    scal_err = scaling_error(W, conv, layer, xs[0], ws[0], S, path, dev) if rank == 0 else None
    # ---------------- e2e through the C ABI with host buffers (pinned), copies inside the region
    e2e = run_e2e(conv, xs, ws, S, stream, n_sets, max(3, min(args.steps, 100)), world, dist if world > 1 else None,
                  dev, job_ops, n_streams=args.e2e_streams)

    if rank == 0:
        peaks = _peaks()
        # the captured shape and variant (int8 F(4x4), target 255; per kernel path)
        full = sh["n"] == layer.n and sh["co"] == layer.c_out and args.alg == "f4" and args.input == "i8" and \
            args.target == 255
        roof = roofline(kern, info, synth.LayerCfg(sh["n"], layer.h, layer.w, layer.c_in, sh["co"], layer.pad),
                        peaks, load_traffic(args.config, "staged" if info.path == 2 else "fused") if full else None)
        path = path_roofline(synth.LayerCfg(sh["n"], layer.h, layer.w, layer.c_in, sh["co"], layer.pad), info,
                             peaks, t_max / args.steps)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_max * 1e3 / args.steps, 5), "higher_is_better": True,
            "scaling": "weak" if args.scaling == "weak" else "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic",
            "config": {
                "workload": f"{cfg.name}: {cfg.description}", "batch_per_gpu": layer.n, "h": layer.h, "w": layer.w,
                "c_in": layer.c_in, "c_out": layer.c_out, "pad": layer.pad, "layout": "NHWC",
                "filter_scaling": layer.scaling, "output": f"int8 requantised (M0=1, S={S})",
                "step": "filter transform + scaling (K1) + conv (" +
                        ("K2, K3F fused GEMM+output per chunk)" if info.path == 1 else "K2,K3,K4 per chunk)"),
                "path": "fused" if info.path == 1 else "staged",
                "input": "uint8, zero points 128 (SURVEY f2)" if u8 else "int8",
                "filter_target_max": args.target if layer.scaling else None,
                "algorithm": "F(2x2,3x3) rational (SURVEY f1)" if info.algorithm == 1 else
                             "F(4x4,3x3) complex (Gaussian integers)",
                "l2": f"inputs/weights/outputs rotated over {n_sets} sets "
                      f"({n_sets * per_set / 2 ** 20:.0f} MiB > 126 MiB L2)",
                "parallelism": f"dp{world} ({'replicated per-rank batches, weak scaling' if args.scaling == 'weak' else sh['mode'] + '-sharded, strong scaling'}; no data-path collective)",
                "chunks": info.n_chunks, "cuda_graph": bool(graphs), "streams": len(lanes),
                "filter_transform_overlapped": bool(args.overlap_filter),
            },
            "roofline": roof["dominant"],
            "path_roofline": path,
            "kernels": roof["all"],
            "kernel_sum_vs_step": round(sum(k["s_per_step"] for k in kern.values()) / (t_max / args.steps), 3),
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e,
            "scaling_error": scal_err,
            "sharded_check": sharded_check,
        }
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours_stack(args):
    """--config C5: the VGG-16 13-layer stack (BASELINE configs[4]) per step:
    13 filter transforms + 13 convs (requantised) + 4 max pools, batch 256 per rank."""
    import torch
    import torch.distributed as dist

    from paper_1901_01965_b200 import _lib as L
    from paper_1901_01965_b200.stack import ConvStack

    rank, local_rank, world = _env_rank()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS["C5"]
    shifts = synth.stack_shifts("C5")
    n = cfg.layers[0].n
    path = {"staged": L.WINO_PATH_STAGED, "fused": L.WINO_PATH_FUSED, "auto": L.WINO_PATH_AUTO}[args.path]
    st = ConvStack(n, cfg.layers, cfg.pools_after, shifts, device=local_rank, path=path)
    n_sets = 2
    xs, wss = [], []
    for i in range(n_sets):
        x, ws = synth.stack_inputs("C5", rank=rank * 1000 + i)
        xs.append(torch.from_numpy(x).to(dev))
        wss.append([torch.from_numpy(w).to(dev) for w in ws])
    stream = torch.cuda.Stream(device=dev)

    def step(j):
        st.transform_filters(wss[j], stream)
        st(xs[j], stream)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i % n_sets)
        stream.synchronize()
        graphs = []
        for j in range(n_sets):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(j)
            graphs.append(g)
        for j in range(3):
            graphs[j % n_sets].replay()
        stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for i in range(args.steps):
                graphs[i % n_sets].replay()
            ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    ops_step = sum(synth.direct_ops(l) for l in cfg.layers)
    value = world * ops_step * args.steps / t_max / 1e12
    # per-layer path roofline summed over the stack
    peaks = _peaks()
    i8 = 2.0 * peaks["bf16_tflops_sustained"] * 1e12
    t_roof = 0.0
    for l, c in zip(cfg.layers, st.convs):
        ops46 = 2 * 46 * c.info.tiles * l.c_in * l.c_out
        byts = c.info.x_bytes + c.info.y_bytes + 92 * l.c_in * l.c_out
        t_roof += max(ops46 / i8, byts / (peaks["hbm_gbs"] * 1e9))
    # roofline of the stack's dominant kernel: every layer's kernels timed alone (as for C2-C4) on the
    # stack's own buffers; the (layer, kernel) with the largest time per step is reported
    kern_l, cur = [], xs[0]
    for i, c in enumerate(st.convs):
        kern_l.append(profile_kernels(c, [cur], [wss[0][i]], [st.outs[i]], shifts[i], stream, 1, 10))
        cur = st.pooled.get(i, st.outs[i])
    dom_l = max(range(len(st.convs)), key=lambda i: max(k["s_per_step"] for k in kern_l[i].values()))
    lay = cfg.layers[dom_l]
    roof = roofline(kern_l[dom_l], st.convs[dom_l].info, synth.LayerCfg(n, lay.h, lay.w, lay.c_in, lay.c_out, lay.pad),
                    peaks, None)
    roof["dominant"]["layer"] = dom_l + 1
    stack_kernel_us = sum(k["s_per_step"] for kl in kern_l for k in kl.values()) * 1e6
    layers_us = [round(sum(k["s_per_step"] for k in kl.values()) * 1e6, 1) for kl in kern_l]
    # e2e: host x in, host final activation out, through the C ABI calls
    xh = xs[0].cpu().pin_memory()
    out = st(xs[0], stream)
    torch.cuda.synchronize()
    yh = torch.empty(out.shape, dtype=torch.int8).pin_memory()
    xd = torch.empty_like(xs[0])
    reps = 3
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(reps):
            xd.copy_(xh, non_blocking=True)
            step_out = None
            st.transform_filters(wss[0], stream)
            step_out = st(xd, stream)
            yh.copy_(step_out, non_blocking=True)
        e1.record(stream)
        stream.synchronize()
    te = e0.elapsed_time(e1) / 1e3
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_max * 1e3 / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"C5: {cfg.description}", "batch_per_gpu": n, "layers": len(cfg.layers),
                       "layout": "NHWC", "filter_scaling": True, "requant_shifts": shifts,
                       "step": "13 filter transforms + 13 convs + 4 max pools",
                       "paths": ["fused" if c.info.path == 1 else "staged" for c in st.convs],
                       "l2": "activations 0.8 GB per layer >> 126 MiB L2; 2 input sets rotated",
                       "parallelism": f"dp{world} (replicated per-rank batches, weak scaling)"},
            "path_roofline": {"t_roof_us": round(t_roof * 1e6, 2), "t_step_us": round(t_max / args.steps * 1e6, 2),
                              "frac": round(t_roof / (t_max / args.steps), 4),
                              "roofline_effective_tops": round(ops_step / t_roof / 1e12, 1)},
            "roofline": roof["dominant"],
            "kernel_sum_vs_step": round(stack_kernel_us / (t_max / args.steps * 1e6), 3),
            "layers_kernel_us": layers_us,
            "gpu_launches": st.launches() * args.steps + len(cfg.layers) * args.steps,
            "clocks": clk.summary(),
            "e2e": {"value": round(world * ops_step * reps / te / 1e12, 3), "unit": "TOPS",
                    "h2d_bytes_per_step": int(xh.numel()), "d2h_bytes_per_step": int(yh.numel()),
                    "steps": reps},
        }
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_stack(shifts)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_stack(shifts):
    import oracle.oracle as O
    O.build()
    cfg = synth.CONFIGS["C5"]
    x, ws = synth.stack_inputs("C5", n=1)
    t0 = time.perf_counter()
    cur = x
    for i, w in enumerate(ws):
        cur = O.wino_conv(cur, w, 1, O.NHWC, scaling=True, M0=1, S=shifts[i]).y8
        if i in cfg.pools_after:
            cur = O.maxpool2(cur, O.NHWC)
    t = time.perf_counter() - t0
    ops = sum(synth.direct_ops(l, n=1) for l in cfg.layers)
    cores = len(os.sched_getaffinity(0))
    return {"value": round(ops / t / 1e12, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
            "sample": f"oracle stack (13 layers + pools) on image 0 of C5 ({ops:.3e} direct ops); {t:.2f} s"}


def scaling_error(W, conv, layer, x, w, S, path, dev, images=4):
    """BASELINE north_star: the scaling-induced error against direct convolution, max-abs and mean-abs
    in output LSBs, on the first `images` images: out32 of the same kernels (an int32-output plan) against
    the exact direct convolution (torch float64 conv2d on the GPU: exact, |sums| < 2^53), and the bench's
    own int8 output against the direct result requantised with the same rule (rha(v / 2^S), clamp)."""
    import torch
    import torch.nn.functional as F
    if not layer.scaling:
        return None
    ne = min(images, x.shape[0])
    xs = x[:ne].contiguous()
    c32 = W.WinoConv2d(ne, layer.h, layer.w, layer.c_in, conv.w_shape[0], layer.pad, W.WINO_NHWC, True,
                       W.WINO_OUT_INT32, device=dev.index, path=path, algorithm=conv.desc.algorithm,
                       input_type=conv.desc.input_type, x_zero_point=conv.desc.x_zero_point,
                       w_zero_point=conv.desc.w_zero_point, filter_target_max=conv.desc.filter_target_max)
    c32.transform_filter(w)
    y32 = c32(xs).long()
    zx, zw = conv.desc.x_zero_point, conv.desc.w_zero_point
    xf = (xs.to(torch.float64) if xs.dtype == torch.int8 else xs.to(torch.float64) - zx).permute(0, 3, 1, 2)
    wf = (w.to(torch.float64) if w.dtype == torch.int8 else w.to(torch.float64) - zw).permute(0, 3, 1, 2)
    ref = F.conv2d(xf, wf, padding=layer.pad).permute(0, 2, 3, 1).round().long()
    conv.transform_filter(w)
    y8 = conv(x, 1, S)[:ne].long()

    def requant(v):
        a = v.abs()
        r = (a + (1 << (S - 1))) >> S if S > 0 else a
        return torch.clamp(torch.where(v < 0, -r, r), -128, 127)

    e32 = (y32 - ref).abs().double()
    e8 = (y8 - requant(ref)).abs().double()
    return {"images": ne, "reference": "direct convolution (torch float64 conv2d, exact)",
            "out32_lsb": {"max_abs": int(e32.max()), "mean_abs": round(float(e32.mean()), 4),
                          "mean_abs_ref": round(float(ref.abs().double().mean()), 2),
                          "mean_rel": round(float(e32.mean() / ref.abs().double().mean()), 6)},
            "y8_lsb": {"max_abs": int(e8.max()), "mean_abs": round(float(e8.mean()), 5),
                       "frac_differing": round(float((e8 > 0).double().mean()), 5), "requant_shift": S}}


def profile_kernels(conv, xs, ws, ys, S, stream, n_sets, reps):
    """Average device duration of each kernel type: for each kernel, a CUDA
    graph of `reps` back-to-back launches of that kernel alone (input/output
    slots rotated as in the timed run, chunks cycled), timed with CUDA events
    on the launching stream; duration = elapsed / reps.  The step's kernel
    sequence adds up to the timed step (checked in the JSON as `sum_vs_step`)."""
    import torch
    from paper_1901_01965_b200 import _lib as L
    info = conv.info
    sp = stream.cuda_stream
    names = {1: "k1_filter", 2: "k2_input", 3: "k3_gemm", 4: "k4_output"} if info.path == 2 else \
        {1: "k1_filter", 2: "k2_input", 3: "k3_fused"}
    w_wino, codes, wsp = conv.w_wino.data_ptr(), conv.codes.data_ptr(), conv.workspace.data_ptr()
    out = {}
    for st in sorted(names):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for r in range(reps):
                j, c = r % n_sets, r % info.n_chunks
                if st == 1:
                    L.wino_transform_filter(conv.plan, ws[j].data_ptr(), w_wino, codes, sp)
                else:
                    L.wino_conv2d_int8_stage(conv.plan, st, c, xs[j].data_ptr(), w_wino, codes, 1, S,
                                             ys[j].data_ptr(), wsp, sp)
        times = []
        with torch.cuda.stream(stream):
            g.replay()
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream); g.replay(); e1.record(stream)
                stream.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3 / reps)
        per_launch = float(np.median(times))
        count = 1 if st == 1 else info.n_chunks
        out[names[st]] = {"s_per_launch": per_launch, "launches_per_step": count, "s_per_step": per_launch * count}
        del g
    return out


def load_traffic(config, path):
    """roofline.traffic: DRAM bytes per launch from the latest committed ncu --set full
    capture of this config and kernel path (profiles/rNN_traffic_<config>_<path>.json, written
    by tools/profile_summary.py), or {} when no capture exists."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          f"r*_traffic_{config}_{path}.json")))
    if not files:
        return {}
    try:
        return json.load(open(files[-1]))["bytes"]
    except Exception:
        return {}


def roofline(kern, info, layer, peaks, traffic=None):
    """Algorithmic work per launch against the measured peaks."""
    T = info.tiles
    chunk_tiles = min(info.chunk_images, layer.n) * info.tiles_h * info.tiles_w
    nch = info.n_chunks
    hbm = peaks["hbm_gbs"]
    i8_sus = 2.0 * peaks["bf16_tflops_sustained"]   # int8 dense = 2 x bf16 (nominal ratio 4.5/2.25)
    px = info.tile * info.tile                     # output pixels per tile (16 F4x4, 4 F2x2)
    mults = alg_mults(info)                        # general multiplications per (tile, cin, cout)
    vpc = 72 if (info.path == 1 and info.algorithm == 0) else 2 * info.planes   # V bytes per (tile, channel)
    x_chunk = chunk_tiles * px * layer.c_in        # ~ bytes of x per chunk
    res = {}
    # K1: reads w (9 Cin Cout B), writes the W' image + codes
    k1_bytes = 9 * layer.c_in * layer.c_out + info.filter_bytes + info.positions * layer.c_out
    # K2: reads x of the chunk, writes V
    k2_bytes = x_chunk + vpc * chunk_tiles * info.cin_pad
    # K3: the method's general multiplies per (tile, cin, cout) (46 = P:228; 16 for F(2x2)), 2 ops each
    k3_ops = 2 * mults * chunk_tiles * layer.c_in * layer.c_out
    k3_bytes = vpc * chunk_tiles * info.cin_pad + info.positions * 4 * chunk_tiles * info.cout_pad + info.filter_bytes
    # K4: reads the M'' int32 per (tile, cout), writes y int8
    k4_bytes = info.positions * 4 * chunk_tiles * layer.c_out + chunk_tiles * px * layer.c_out
    # K3F (fused): the K3 work; bytes: V once, W' once, y int8 once
    k3f_bytes = vpc * chunk_tiles * info.cin_pad + info.filter_bytes + chunk_tiles * px * layer.c_out
    # The GEMM kernel has two roofs: its algorithmic int ops against the int8 tensor peak, and its own
    # HBM bytes (V in, W' in, M'' or y out) against the HBM peak.  The binding roof is the one with the
    # larger minimum time (the kernel's arithmetic intensity against the ridge point); the bench line
    # reports that one and keeps the other as a second view.
    gemm = "k3_gemm" if info.path == 2 else "k3_fused"
    if info.path != 2:
        k3_bytes = k3f_bytes
    t_tc, t_hbm = k3_ops / (i8_sus * 1e12), k3_bytes / (hbm * 1e9)
    gemm_spec = ("hbm", k3_bytes, hbm, "GB/s") if t_hbm >= t_tc else ("tensor", k3_ops, i8_sus, "TOPS")
    spec = {"k1_filter": ("hbm", k1_bytes, hbm, "GB/s"), "k2_input": ("hbm", k2_bytes, hbm, "GB/s"), gemm: gemm_spec}
    if info.path == 2:
        spec["k4_output"] = ("hbm", k4_bytes, hbm, "GB/s")
    all_k = {}
    for name, (bound, work, peak, unit) in spec.items():
        t = kern[name]["s_per_launch"]
        achieved = work / t / (1e9 if unit == "GB/s" else 1e12)
        d = {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": unit,
             "frac": round(achieved / peak, 4), "traffic": (traffic or {}).get(name), "us_per_launch": round(t * 1e6, 3),
             "launches_per_step": kern[name]["launches_per_step"],
             "share_of_step": None, "algorithmic_per_launch": work}
        if name == gemm:
            d["roof_times_us"] = {"tensor": round(t_tc * 1e6, 3), "hbm": round(t_hbm * 1e6, 3)}
            d["tensor_view"] = {"int_ops_per_launch": k3_ops, "achieved_tops": round(k3_ops / t / 1e12, 2),
                                "peak_tops": round(i8_sus, 1), "frac": round(k3_ops / t / 1e12 / i8_sus, 4)}
            d["hbm_view"] = {"bytes_per_launch": k3_bytes, "achieved_gbs": round(k3_bytes / t / 1e9, 1),
                             "frac_of_hbm": round(k3_bytes / t / 1e9 / hbm, 4)}
        all_k[name] = d
    tot = sum(kern[k]["s_per_step"] for k in kern)
    for k in all_k:
        all_k[k]["share_of_step"] = round(kern[k]["s_per_step"] / tot, 4)
    dom = max(all_k, key=lambda k: kern[k]["s_per_step"])
    dominant = dict(all_k[dom]); dominant["kernel"] = dom
    dominant["peak_source"] = peaks["source"] + (
        "; int8 = 2 x bf16 sustained" if dominant["bound"] == "tensor" else "; hbm_gbs")
    return {"dominant": dominant, "all": all_k}


def alg_mults(info):
    """The method's general multiplications per (tile, input channel, output channel): 46 for the
    complex F(4x4) (the fused path's 4-multiplication form is an implementation choice), 16 for
    the rational F(2x2)."""
    return 16 if info.algorithm == 1 else 46


def path_roofline(layer, info, peaks, t_step):
    """t_roof = max(2*mults*T*Cin*Cout / P_int8, (x + y + W') / HBM) for one
    rank's step, and the achieved fraction of it."""
    T = info.tiles
    ops46 = 2 * alg_mults(info) * T * layer.c_in * layer.c_out
    byts = info.x_bytes + info.y_bytes + info.filter_bytes + 9 * layer.c_in * layer.c_out
    i8 = 2.0 * peaks["bf16_tflops_sustained"] * 1e12
    t_roof = max(ops46 / i8, byts / (peaks["hbm_gbs"] * 1e9))
    return {"t_roof_us": round(t_roof * 1e6, 3), "t_step_us": round(t_step * 1e6, 3),
            "frac": round(t_roof / t_step, 4), "bound": "tensor" if ops46 / i8 > byts / (peaks["hbm_gbs"] * 1e9)
            else "hbm", "roofline_effective_tops": round(synth.direct_ops(layer) / t_roof / 1e12, 1)}


def run_e2e(conv, xs, ws, S, stream, n_sets, reps, world, dist, dev, job_ops, n_streams=3):
    """Same metric through the C ABI with HOST buffers: every step copies x and w
    from pinned host memory, runs K1..K4 (wino_transform_filter +
    wino_conv2d_int8_host, whose H2D / D2H copies are inside the call) and reads
    y back to pinned host memory.  Steps rotate over `n_streams` streams, each
    with its own device buffers, so one step's copies overlap another's compute
    (how a user pipelines the API)."""
    import torch
    from paper_1901_01965_b200 import _lib as L
    info = conv.info
    k = min(n_sets, 8)
    xh = [xs[i].cpu().pin_memory() for i in range(k)]
    wh = [ws[i].cpu().pin_memory() for i in range(k)]
    yh = [torch.empty(conv.y_shape, dtype=torch.int8).pin_memory() for _ in range(k)]
    lanes = []
    for si in range(n_streams):
        st = stream if si == 0 else torch.cuda.Stream(device=dev)
        lanes.append({
            "st": st, "sp": st.cuda_stream,
            "xd": torch.empty(conv.x_shape, dtype=torch.int8, device=dev),
            "yd": torch.empty(conv.y_shape, dtype=torch.int8, device=dev),
            "wd": torch.empty(conv.w_shape, dtype=torch.int8, device=dev),
            "ww": conv.w_wino if si == 0 else torch.empty_like(conv.w_wino),
            "cd": conv.codes if si == 0 else torch.empty_like(conv.codes),
            "ws": conv.workspace if si == 0 else torch.empty_like(conv.workspace),
        })

    def step(i):
        j, ln = i % k, lanes[i % n_streams]
        with torch.cuda.stream(ln["st"]):
            ln["wd"].copy_(wh[j], non_blocking=True)
        L.wino_transform_filter(conv.plan, ln["wd"].data_ptr(), ln["ww"].data_ptr(), ln["cd"].data_ptr(), ln["sp"])
        L.wino_conv2d_int8_host(conv.plan, xh[j].data_ptr(), ln["ww"].data_ptr(), ln["cd"].data_ptr(), 1, S,
                                yh[j].data_ptr(), ln["xd"].data_ptr(), ln["yd"].data_ptr(), ln["ws"].data_ptr(),
                                ln["sp"])

    for i in range(3 * n_streams):
        step(i)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for ln in lanes[1:]:
        ln["st"].wait_event(e0)
    h0 = time.perf_counter()
    for i in range(reps):
        step(i)
    host_issue = (time.perf_counter() - h0) / reps
    for ln in lanes[1:]:
        ev = torch.cuda.Event()
        ev.record(ln["st"])
        stream.wait_event(ev)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    v = job_ops * reps / float(t.item()) / 1e12
    return {"value": round(v, 3), "unit": "TOPS", "h2d_bytes_per_step": int(info.x_bytes + np.prod(conv.w_shape)),
            "d2h_bytes_per_step": int(info.y_bytes), "steps": reps, "streams": n_streams,
            "ms_per_step": round(float(t.item()) * 1e3 / reps, 4), "host_issue_ms_per_step": round(host_issue * 1e3, 4)}


# ----------------------------------------------------------------------------- CPU oracle arm
def _oracle_sample(config, budget_s):
    """A bounded sample of the workload for the CPU oracle: the first `rows`
    output rows of one image (pad 1), sized to ~budget_s seconds."""
    from oracle import oracle as O
    layer = synth.CONFIGS[config].layers[0]
    x, w = synth.config_inputs(config, n=1)
    S = synth.requant_shift(layer)

    def run(rows):
        xs = np.ascontiguousarray(x[:, :rows])
        t0 = time.perf_counter()
        O.wino_conv(xs, w, layer.pad, O.NHWC, scaling=layer.scaling, M0=1, S=S)
        return time.perf_counter() - t0

    rows = min(layer.h, 4)
    dt = run(rows)
    while rows < layer.h and dt < budget_s / 3:
        rows = min(layer.h, rows * 2)
        dt = run(rows)
    ops = synth.direct_ops(synth.LayerCfg(1, rows, layer.w, layer.c_in, layer.c_out, layer.pad))
    return run, rows, ops, dt


def cpu_baseline(config, budget_s=10.0):
    import oracle.oracle as O
    O.build()
    run, rows, ops, _ = _oracle_sample(config, budget_s / 2)
    reps, t = 0, 0.0
    while t < budget_s / 2 or reps < 1:
        t += run(rows); reps += 1
    cores = len(os.sched_getaffinity(0))
    return {"value": round(ops * reps / t / 1e12, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
            "sample": f"oracle.wino_conv (plain C, OpenMP {cores} threads) on image 0 rows 0..{rows - 1} "
                      f"of {config} ({ops:.3e} direct ops) x {reps}; {t:.2f} s"}


def run_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return
    import oracle.oracle as O
    O.build()
    per_step_budget = max(0.05, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    run, rows, ops, _ = _oracle_sample(args.config, per_step_budget)
    for _ in range(args.warmup):
        run(rows)
    t = 0.0
    for _ in range(args.steps):
        t += run(rows)
    v = ops * args.steps / t / 1e12
    cores = len(os.sched_getaffinity(0))
    layer = synth.CONFIGS[args.config].layers[0]
    cfg = synth.CONFIGS[args.config]
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3 / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.description}", "batch_per_gpu": layer.n, "h": layer.h,
                       "w": layer.w, "c_in": layer.c_in, "c_out": layer.c_out, "layout": "NHWC",
                       "filter_scaling": layer.scaling},
            "cpu_baseline": {"value": round(v, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
                             "sample": f"per step: oracle.wino_conv on image 0 rows 0..{rows - 1} "
                                       f"({ops:.3e} direct ops)"},
            "e2e": {"value": round(v, 6), "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--streams", type=int, default=3,
                    help="independent batches in flight on separate streams (own filter/workspace buffers)")
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "staged"],
                    help="auto: the plan picks fused for c_in <= 256 (C2-C4, C5 layers 1-8), staged otherwise")
    ap.add_argument("--input", default="i8", choices=["i8", "u8"],
                    help="u8: uint8 tensors with zero points (SURVEY f2; either algorithm and path, c_in <= 224)")
    ap.add_argument("--alg", default="f4", choices=["f4", "f2"],
                    help="f4: complex F(4x4,3x3) (the north star); f2: rational F(2x2,3x3) (SURVEY f1, either path)")
    ap.add_argument("--target", type=int, default=255, choices=[255, 127],
                    help="filter scaling target: 255 = the paper's (two-piece W'); 127 = int8-native single-piece "
                         "W' (SURVEY f3, staged F(4x4) int8)")
    ap.add_argument("--overlap-filter", type=int, default=0,
                    help="1: filter transform on a side stream concurrent with the input transform")
    ap.add_argument("--e2e-streams", type=int, default=3,
                    help="host-buffer (e2e) leg: steps in flight on separate streams, so copies overlap compute")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=24.0,
                    help="CPU oracle baseline budget (about half of it is the timed sample)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "C5":
        run_ours_stack(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
