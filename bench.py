"""Benchmark of the complex-Winograd int8 3x3 conv hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

One step = the whole hot path over one batch of
synthetic input.  Default workload: C5 (BASELINE.json configs[4]), the largest
configuration that fits one GPU -- the VGG-16 13-layer stack at 224x224, batch
256: per layer the filter transform + scaling (K1) and the convolution (K2
input transform -> K3F fused tcgen05 GEMMs + reverse scaling + output
transform, or K2 -> K3 -> K4 staged, per WINO_PATH_AUTO), requantised, with
the 2x2 max pools.  C1-C4 are single layers (`--config`).

Multi-GPU (BASELINE north_star): `--gpus N` partitions the
configured batch over N ranks (and Cout for batch 1) with no collective on the
data path -- one process per GPU; when WORLD_SIZE is unset the script re-runs
itself under `torch.distributed.run` with N ranks.  NCCL carries only the
barrier, the max-over-ranks reduction of the timed region and the gather of
the outputs for checking (outside the timed region).

Timing: CUDA graphs, W warm-up steps, then exactly K steps
bracketed by a barrier and a device synchronisation, CUDA events on the
launching stream, max over ranks; then 5 trials of R steps (R so that a trial
is >= 100 ms) with their median and minimum; K1 (offline in the paper)
is also timed separately and the step without it reported.  Activations are
larger than the 126 MiB L2 (or rotated over enough input sets).

`--impl reference` times the CPU oracle (oracle/, plain C) on the host cores,
one bounded sample of the same workload per step.
`--plan-only` (CPU, gloo) spawns the ranks and prints their shards only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "int8 3x3 conv effective TOPS (direct-conv ops/s)"
L2_BYTES = 126 * 2 ** 20
DEFAULT_STEPS = {"C1": 2000, "C2": 2000, "C3": 2000, "C4": 1000, "C5": 50}


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def _peaks():
    """Roofline denominators: MEASURED_PEAKS.json (driver-measured HBM copy bandwidth and cuBLAS bf16,
    burst and sustained); int8 = 2 x bf16 (the nominal ratio 4.5 / 2.25 PFLOP/s, B200_PROFILING.md).
    Kernels timed alone are compared with the burst figures."""
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16 = float(p.get("bf16_tflops", 1590.0))
    return {
        "hbm_gbs": float(p.get("hbm_gbs", 6650.0)),
        "int8_tops_burst": 2.0 * bf16,
        "int8_tops_sustained": 2.0 * float(p.get("bf16_tflops_sustained", 1400.0)),
        "int8_tops_nominal": 4500.0,
        "source": "MEASURED_PEAKS.json (measured)" if p else "B200_PROFILING.md fallback",
    }


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


# ----------------------------------------------------------------------------- ranks
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn_ranks(args):
    """`--gpus N` with no WORLD_SIZE in the environment: re-run this script under torch.distributed.run
    with N ranks on 127.0.0.1 (the driver's own launch line), and exit with its status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _phase(name):
    """WINO_BENCH_TRACE=1: per-rank progress on stderr (debugging multi-rank runs)."""
    if os.environ.get("WINO_BENCH_TRACE"):
        print(f"[rank {os.environ.get('RANK', 0)}] {time.strftime('%H:%M:%S')} {name}", file=sys.stderr, flush=True)


def _device_index(local_rank):
    """This rank's GPU: LOCAL_RANK, or round-robin over the visible GPUs in the gloo validation mode."""
    import torch
    if os.environ.get("WINO_DIST_BACKEND", "nccl") == "gloo":
        return local_rank % max(1, torch.cuda.device_count())
    return local_rank


def _init_dist(world, local_rank, backend="nccl"):
    """The process group of a multi-rank run (None at world size 1).  WINO_DIST_BACKEND=gloo replaces NCCL
    (a validation mode: with fewer GPUs than ranks, ranks share devices round-robin; the path has no
    data-path collective, so their kernels never wait on one another -- timings are then not per-GPU)."""
    import torch
    import torch.distributed as dist
    backend = os.environ.get("WINO_DIST_BACKEND", backend)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    return dist if world > 1 else None


def _shard(args, n, c_out, world, rank):
    from paper_1901_01965_b200 import shard as SH
    if args.scaling == "strong":
        return SH.shard(n, c_out, world, rank)
    return {"mode": "replica", "n0": 0, "n": n, "co0": 0, "co": c_out}


def run_plan_only(args):
    """CPU (gloo) view of the multi-GPU launch: every rank computes its shard of the configuration and
    gathers stand-in outputs (filled with rank + 1) through the same checking gather the GPU run uses
    (empty shards included); rank 0 prints the shards.  Used by tests/test_multi_gloo.py."""
    import torch
    from paper_1901_01965_b200 import shard as SH
    rank, local_rank, world = _env_rank()
    dist = _init_dist(world, local_rank, "gloo")
    cfg = synth.CONFIGS[args.config]
    layer = cfg.layers[0]
    sh = _shard(args, layer.n, layer.c_out, world, rank)
    ho, wo = layer.h + 2 * layer.pad - 2, layer.w + 2 * layer.pad - 2
    local = torch.full((sh["n"], ho, wo, sh["co"]), rank + 1, dtype=torch.int8)
    if world > 1:
        gathered = SH.gather_nhwc(local, (layer.n, ho, wo, layer.c_out), sh, world)
        shards = [None] * world
        dist.all_gather_object(shards, sh)
    else:
        gathered, shards = local, [sh]
    t = SH.max_over_ranks(0.25 * (rank + 1))
    if rank == 0:
        owner = gathered.to(torch.int64)
        per_rank = [int((owner == r + 1).sum()) for r in range(world)]
        print(json.dumps({"plan_only": True, "config": args.config, "world": world, "shards": shards,
                          "gathered_shape": list(gathered.shape), "elements_per_rank": per_rank,
                          "max_over_ranks": t, "torchrun": "TORCHELASTIC_RUN_ID" in os.environ}), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- roofline
def conv_alg(info, c_in, c_out, images=None):
    """SURVEY 8(d) algorithmic work of one conv (or of `images` of its batch): 2 x 46 general
    multiplications per (tile, c_in, c_out) (16 for F(2x2)), and x read once + y written once +
    W' read once (92 B per (c_in, c_out) for F(4x4): 46 planes x 2 pieces; 32 for F(2x2))."""
    mults = 16 if info.algorithm == 1 else 46
    n_img = info.tiles // (info.tiles_h * info.tiles_w)
    frac = 1.0 if images is None else images / n_img
    tiles = info.tiles * frac
    ops = 2 * mults * tiles * c_in * c_out
    byts = (info.x_bytes + info.y_bytes) * frac + 2 * mults * c_in * c_out
    return ops, byts


def conv_roof_s(info, c_in, c_out, peaks, images=None, peak_key="int8_tops_burst"):
    ops, byts = conv_alg(info, c_in, c_out, images)
    return max(ops / (peaks[peak_key] * 1e12), byts / (peaks["hbm_gbs"] * 1e9)), ops, byts


def design_bytes(name, info, c_in, c_out, images):
    """Bytes the kernel of THIS design moves per launch (V, M'' and W' images included): the build's own
    traffic, reported beside the algorithmic figure."""
    n_img = info.tiles // (info.tiles_h * info.tiles_w)
    tiles = info.tiles * images / n_img
    x = info.x_bytes * images / n_img
    y = info.y_bytes * images / n_img
    vpc = 72 if (info.path == 1 and info.algorithm == 0) else 2 * info.planes
    v = vpc * tiles * info.cin_pad
    m = info.positions * 4 * tiles * info.cout_pad
    return {"k1_filter": 9 * c_in * c_out + info.filter_bytes + info.codes_bytes,
            "k2_input": x + v, "k3_fused": v + info.filter_bytes + y,
            "k3_gemm": v + info.filter_bytes + m, "k4_output": m + y}[name]


def kernel_roofline(name, kern, info, c_in, c_out, peaks, chunk_images):
    """Roofline object of one kernel: its share of the conv's SURVEY 8(d) algorithmic work per launch
    (the GEMM-carrying kernel: the whole conv's x + y + W' bytes and 2 x 46 ops per (tile, cin, cout),
    whichever roof binds; K2: the x bytes it reads; K4: the y bytes it writes; K1: w + the W' image)
    against the burst peaks (kernels timed alone)."""
    t = kern[name]["s_per_launch"]
    ops, byts = conv_alg(info, c_in, c_out, chunk_images)
    n_img = info.tiles // (info.tiles_h * info.tiles_w)
    t_tc = t_hbm = None
    if name in ("k3_fused", "k3_gemm"):
        t_tc, t_hbm = ops / (peaks["int8_tops_burst"] * 1e12), byts / (peaks["hbm_gbs"] * 1e9)
        bound = "tensor" if t_tc > t_hbm else "hbm"
        work = ops if bound == "tensor" else byts
    elif name == "k2_input":
        bound, work = "hbm", info.x_bytes * chunk_images / n_img
    elif name == "k4_output":
        bound, work = "hbm", info.y_bytes * chunk_images / n_img
    else:
        bound, work = "hbm", 9 * c_in * c_out + 2 * (16 if info.algorithm == 1 else 46) * c_in * c_out
    if bound == "tensor":
        achieved, peak, unit = work / t / 1e12, peaks["int8_tops_burst"], "TOPS"
    else:
        achieved, peak, unit = work / t / 1e9, peaks["hbm_gbs"], "GB/s"
    own = design_bytes(name, info, c_in, c_out, chunk_images)
    d = {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 1), "unit": unit,
         "frac": round(achieved / peak, 4), "traffic": None, "kernel": name,
         "us_per_launch": round(t * 1e6, 3), "launches_per_step": kern[name]["launches_per_step"],
         "algorithmic_per_launch": round(work), "design_bytes_per_launch": round(own),
         "design_bytes_vs_algorithmic_bytes": round(own / max(1.0, byts if name.startswith("k3") else work), 2)}
    if t_tc is not None:
        d["roof_times_us"] = {"tensor": round(t_tc * 1e6, 3), "hbm": round(t_hbm * 1e6, 3)}
        d["tensor_view"] = {"alg_int_ops_per_launch": round(ops), "achieved_tops": round(ops / t / 1e12, 2),
                            "peak_tops": round(peaks["int8_tops_burst"], 1),
                            "frac": round(ops / t / 1e12 / peaks["int8_tops_burst"], 4)}
    return d


def load_traffic(tag):
    """roofline.traffic: DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the
    latest committed ncu --set full capture summary profiles/rNN_traffic_<tag>.json, or {}."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_traffic_{tag}.json")))
    if not files:
        return {}
    try:
        return json.load(open(files[-1]))["bytes"]
    except Exception:
        return {}


# ----------------------------------------------------------------------------- timing helpers
def _timed(stream_list, fn, dist, dev):
    """Barrier + synchronise, CUDA events on stream_list[0] around fn(), synchronise + barrier;
    returns the max over ranks of the elapsed seconds."""
    import torch
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    main = stream_list[0]
    ev0.record(main)
    for st_ in stream_list[1:]:
        st_.wait_event(ev0)
    fn()
    for st_ in stream_list[1:]:
        e_ = torch.cuda.Event()
        e_.record(st_)
        main.wait_event(e_)
    ev1.record(main)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1) / 1e3], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _trials(run, per_step_s, job_ops, dist, streams, dev, n_trials=5, min_s=0.1):
    """n_trials trials of R steps, R chosen so a trial lasts >= min_s; median and min."""
    reps = max(1, math.ceil(min_s / max(per_step_s, 1e-9)))
    vals = []
    for _ in range(n_trials):
        t = _timed(streams, lambda: run(reps), dist, dev)
        vals.append(job_ops * reps / t / 1e12)
    return {"trials": n_trials, "steps_per_trial": reps, "tops": [round(v, 3) for v in vals],
            "median_tops": round(float(np.median(vals)), 3), "min_tops": round(float(np.min(vals)), 3),
            "max_tops": round(float(np.max(vals)), 3)}


def profile_kernels(conv, xs, ws, ys, S, stream, n_sets, reps, lanes=1):
    """Average device duration of each kernel type: for each kernel, a CUDA graph of `reps` launches of
    that kernel alone (input/output slots rotated, chunks cycled), spread round-robin over `lanes` streams
    forked from `stream` as the timed run overlaps them (1 = back to back on one stream), timed with CUDA
    events on `stream`; duration = elapsed / reps (median of 3)."""
    import torch
    from paper_1901_01965_b200 import _lib as L
    info = conv.info
    names = {1: "k1_filter", 2: "k2_input", 3: "k3_gemm", 4: "k4_output"} if info.path == L.WINO_PATH_STAGED \
        else {1: "k1_filter", 2: "k2_input", 3: "k3_fused"}
    w_wino, codes, wsp = conv.w_wino.data_ptr(), conv.codes.data_ptr(), conv.workspace.data_ptr()
    lanes = max(1, min(lanes, info.lanes if info.lanes > 1 else lanes))
    aux = [stream] + [torch.cuda.Stream(device=stream.device) for _ in range(lanes - 1)]
    out = {}
    for st in sorted(names):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fork = torch.cuda.Event()
            fork.record(stream)
            for a in aux[1:]:
                a.wait_event(fork)
            for r in range(reps):
                j, c = r % n_sets, r % info.n_chunks
                # a chunk's V buffer belongs to lane c % info.lanes: keep chunks of one buffer on one stream
                sp = aux[(c if info.lanes > 1 else r) % lanes].cuda_stream
                if st == 1:
                    sp = aux[r % lanes].cuda_stream
                    L.wino_transform_filter(conv.plan, ws[j].data_ptr(), w_wino, codes, sp)
                else:
                    L.wino_conv2d_int8_stage(conv.plan, st, c, xs[j].data_ptr(), w_wino, codes, 1, S,
                                             ys[j].data_ptr(), wsp, sp)
            for a in aux[1:]:
                e_ = torch.cuda.Event()
                e_.record(a)
                stream.wait_event(e_)
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


# ----------------------------------------------------------------------------- GPU arm, one layer (C1-C4)
def run_ours(args):
    import torch

    layer0 = synth.CONFIGS[args.config].layers[0]
    if args.input == "u8" and layer0.c_in > 224:   # the plan would refuse it (WINO_ERR_UNSUPPORTED)
        if int(os.environ.get("RANK", 0)) == 0:
            print(json.dumps({"metric": METRIC, "config": {"workload": args.config, "input": "u8"},
                              "unsupported": f"uint8 input needs c_in <= 224 (int32 exactness of the int9 values, "
                                             f"DESIGN.md A28); {args.config} has c_in = {layer0.c_in}"}), flush=True)
        return

    import paper_1901_01965_b200 as W
    from paper_1901_01965_b200 import _lib as L
    from paper_1901_01965_b200 import shard as SH

    rank, local_rank, world = _env_rank()
    dist = _init_dist(world, local_rank)
    local_rank = _device_index(local_rank)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS[args.config]
    layer = cfg.layers[0]
    S = synth.requant_shift(layer)
    sh = _shard(args, layer.n, layer.c_out, world, rank)
    empty = sh["n"] == 0 or sh["co"] == 0        # e.g. C1 (Cout 4) at 8 ranks: nothing to launch
    path = {"staged": W.WINO_PATH_STAGED, "fused": W.WINO_PATH_FUSED, "auto": W.WINO_PATH_AUTO}[args.path]
    alg = W.WINO_ALG_F2X2 if args.alg == "f2" else W.WINO_ALG_F4X4
    u8 = args.input == "u8"           # --input u8: the same values as uint8 with zero points 128
    zp = 128 if u8 else 0
    to_in = (lambda a: (a.astype(np.int16) + 128).astype(np.uint8)) if u8 else (lambda a: a)
    mk = dict(device=local_rank, path=path, algorithm=alg, input_type=W.WINO_IN_UINT8 if u8 else W.WINO_IN_INT8,
              x_zero_point=zp, w_zero_point=zp, filter_target_max=args.target)
    ops_local = synth.direct_ops(synth.LayerCfg(sh["n"], layer.h, layer.w, layer.c_in, sh["co"], layer.pad))
    job_ops = synth.direct_ops(layer) * (world if args.scaling == "weak" else 1)
    xs, ws, ys, lanes, graphs, graphs_nok1 = [], [], [], [], {}, {}
    conv = None
    n_sets = 1
    l2_label = "empty shard on rank 0"
    if not empty:
        conv = W.WinoConv2d(sh["n"], layer.h, layer.w, layer.c_in, sh["co"], layer.pad, W.WINO_NHWC, layer.scaling,
                            W.WINO_OUT_INT8, **mk)
        info = conv.info
        per_set = info.x_bytes + sh["co"] * 9 * layer.c_in + info.y_bytes
        # rotate enough input sets to exceed L2; capped at 64 (C1, the parity-size case, and its Cout shards
        # would need thousands -- each one a captured graph per lane): those runs are labelled L2-resident
        n_sets = min(64, max(2, math.ceil(1.2 * L2_BYTES / per_set)))
        l2_label = (f"inputs/weights/outputs rotated over {n_sets} sets (> 126 MiB L2)" if n_sets * per_set > L2_BYTES
                    else f"{n_sets} input sets of {per_set} B: L2-resident (parity-size config, not a bench line)")
        for i in range(n_sets):
            # global tensors of set i (the seeded config for i = 0), this rank's slice
            x, w = synth.config_inputs(args.config, rank=i if args.scaling == "strong" else rank * 1000 + i)
            if args.scaling == "strong":
                x = x[sh["n0"]: sh["n0"] + sh["n"]]
                w = w[sh["co0"]: sh["co0"] + sh["co"]]
            xs.append(torch.from_numpy(np.ascontiguousarray(to_in(x))).to(dev))
            ws.append(torch.from_numpy(np.ascontiguousarray(to_in(w))).to(dev))
            ys.append(torch.empty(conv.y_shape, dtype=torch.int8, device=dev))
        stream = torch.cuda.Stream(device=dev)
        # independent batches in flight on `--streams` streams, each with its own W'/codes/workspace
        lanes = [(stream, conv.w_wino, conv.codes, conv.workspace)]
        for _ in range(1, max(1, args.streams)):
            lanes.append((torch.cuda.Stream(device=dev), torch.empty_like(conv.w_wino), torch.empty_like(conv.codes),
                          torch.empty_like(conv.workspace)))
        streams = [ln[0] for ln in lanes]

        def step(j, lane=0, k1=True):
            st_, ww_, cd_, ws_ = lanes[lane]
            if k1:
                L.wino_transform_filter(conv.plan, ws[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), st_.cuda_stream)
            L.wino_conv2d_int8(conv.plan, xs[j].data_ptr(), ww_.data_ptr(), cd_.data_ptr(), 1, S, ys[j].data_ptr(),
                               ws_.data_ptr(), st_.cuda_stream)

        with torch.cuda.stream(stream):
            for ln in range(len(lanes)):            # every lane's codes seen once, outside the graphs
                step(0, ln)
            for i in range(args.warmup):
                step(i % n_sets, i % len(lanes))
            torch.cuda.synchronize()
            for ln, (st_, _, _, _) in enumerate(lanes):
                with torch.cuda.stream(st_):
                    for j in range(n_sets):
                        for k1, gd in ((True, graphs), (False, graphs_nok1)):
                            g = torch.cuda.CUDAGraph()
                            with torch.cuda.graph(g, stream=st_):
                                step(j, ln, k1)
                            gd[(ln, j)] = g
                    for j in range(max(args.warmup, 3)):
                        graphs[(ln, j % n_sets)].replay()
            torch.cuda.synchronize()

        def run_steps(k, gd=graphs, n_l=None):
            n_l = n_l or len(lanes)
            for i in range(k):
                ln = i % n_l
                with torch.cuda.stream(lanes[ln][0]):
                    gd[(ln, i % n_sets)].replay()
    else:
        streams = [torch.cuda.Stream(device=dev)]

        def run_steps(k, gd=None, n_l=None):
            return None

    launches_per_step = 0 if empty else 1 + conv.info.stages * conv.info.n_chunks
    _phase("timed")
    # ---------------- the timed region: exactly K steps
    with ClockSampler(local_rank) as clk:
        t_max = _timed(streams, lambda: run_steps(args.steps), dist, dev)
    value = job_ops * args.steps / t_max / 1e12
    per_step = t_max / args.steps
    _phase("trials")
    # ---------------- outside the timed region: trials, K1 split, single-stream latency
    trials = _trials(run_steps, per_step, job_ops, dist, streams, dev)
    t_nok1 = _timed(streams, lambda: run_steps(args.steps, graphs_nok1), dist, dev)
    n_single = max(20, args.steps // 10)
    t_single = _timed(streams[:1], lambda: run_steps(n_single, graphs, 1), dist, dev)
    single_ms = t_single * 1e3 / n_single
    _phase("profile")
    kern = profile_kernels(conv, xs, ws, ys, S, streams[0], n_sets, 60) if not empty else {}
    # ---------------- self-check of the timed graphs' output: set 0 (lane 0), this rank's first image
    self_check = None
    if not empty:
        graphs[(0, 0)].replay()
        torch.cuda.synchronize()
        if rank == 0:
            self_check = _self_check_layer(args, layer, sh, ys[0], S, u8, zp)
    _phase("gather")
    # ---------------- partitioned runs: gather the outputs of set 0 (checking only) and compare them with
    # rank 0's single-GPU run of the whole problem
    sharded_check = None
    if world > 1 and args.scaling == "strong":
        ho, wo = layer.h + 2 * layer.pad - 2, layer.w + 2 * layer.pad - 2
        y_loc = ys[0] if not empty else torch.zeros((sh["n"], ho, wo, sh["co"]), dtype=torch.int8, device=dev)
        y_all = SH.gather_nhwc(y_loc, (layer.n, ho, wo, layer.c_out), sh, world, dev)
        n_empty = torch.tensor([1 if empty else 0], device=dev)
        dist.all_reduce(n_empty)
        if rank == 0:
            xf, wf = synth.config_inputs(args.config, rank=0)
            cf = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, layer.pad, W.WINO_NHWC,
                              layer.scaling, W.WINO_OUT_INT8, **mk)
            cf.transform_filter(torch.from_numpy(np.ascontiguousarray(to_in(wf))).to(dev))
            y_one = cf(torch.from_numpy(np.ascontiguousarray(to_in(xf))).to(dev), 1, S)
            sharded_check = {"mode": sh["mode"], "gathered_bytes": int(y_all.numel()),
                             "empty_ranks": int(n_empty.item()),
                             "collective": f"all_gather_into_tensor ({dist.get_backend()}), checking only",
                             "equal_to_single_gpu": bool(torch.equal(y_all, y_one))}
    _phase("e2e")
    scal_err = scaling_error(W, conv, layer, xs[0], ws[0], S, path, dev) if rank == 0 and not empty else None
    e2e = run_e2e(conv, xs, ws, S, streams[0], n_sets, max(3, min(args.steps, 100)), dist, dev, job_ops, empty,
                  n_streams=args.e2e_streams)

    if rank == 0:
        peaks = _peaks()
        info = conv.info
        chunk_imgs = min(info.chunk_images, sh["n"])
        all_k = {k: kernel_roofline(k, kern, info, layer.c_in, sh["co"], peaks, chunk_imgs) for k in kern}
        tot = sum(kern[k]["s_per_step"] for k in kern)
        for k in all_k:
            all_k[k]["share_of_step"] = round(kern[k]["s_per_step"] / tot, 4)
        dom = max(all_k, key=lambda k: kern[k]["s_per_step"])
        roof = dict(all_k[dom])
        full = sh["n"] == layer.n and sh["co"] == layer.c_out and args.alg == "f4" and not u8 and args.target == 255
        if full:
            tag = f"{args.config}_{'staged' if info.path == W.WINO_PATH_STAGED else 'fused'}"
            roof["traffic"] = load_traffic(tag).get(dom)
        roof["peak_source"] = peaks["source"] + (" (int8 = 2 x bf16 burst)" if roof["bound"] == "tensor"
                                                 else " (hbm_gbs, burst copy)")
        t_roof, ops46, byts = conv_roof_s(info, layer.c_in, sh["co"], peaks)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 5), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {
                "workload": f"{cfg.name}: {cfg.description}", "batch": layer.n, "batch_per_gpu": sh["n"],
                "h": layer.h, "w": layer.w, "c_in": layer.c_in, "c_out": layer.c_out, "c_out_per_gpu": sh["co"],
                "pad": layer.pad, "layout": "NHWC", "filter_scaling": layer.scaling,
                "output": f"int8 requantised (M0=1, S={S})",
                "step": "filter transform + scaling (K1) + conv (" +
                        ("K2, K3F fused GEMM+output per chunk)" if info.path == W.WINO_PATH_FUSED
                         else "K2,K3,K4 per chunk)"),
                "path": "fused" if info.path == W.WINO_PATH_FUSED else "staged",
                "input": "uint8, zero points 128 (SURVEY f2)" if u8 else "int8",
                "filter_target_max": args.target if layer.scaling else None,
                "algorithm": "F(2x2,3x3) rational (SURVEY f1)" if info.algorithm == 1 else
                             "F(4x4,3x3) complex (Gaussian integers)",
                "l2": l2_label,
                "parallelism": f"dp{world}: " + (f"{sh['mode']}-partitioned (strong scaling)" if args.scaling == "strong"
                                                 else "replicated per-rank batches (weak scaling)") +
                               "; no data-path collective",
                "chunks": info.n_chunks, "cuda_graph": True, "streams": len(lanes),
            },
            "roofline": roof,
            "path_roofline": {"t_roof_us": round(t_roof * 1e6, 3), "t_step_us": round(per_step * 1e6, 3),
                              "frac": round(t_roof / per_step, 4),
                              "bound": "tensor" if ops46 / peaks["int8_tops_burst"] / 1e12 >
                                       byts / peaks["hbm_gbs"] / 1e9 else "hbm",
                              "alg_int_ops": round(ops46), "alg_bytes": round(byts),
                              "roofline_effective_tops": round(ops_local / t_roof / 1e12, 1)},
            "kernels": all_k,
            "kernel_sum_vs_step": round(tot / per_step, 3),
            "trials": trials,
            "k1": {"us_per_step": round(kern["k1_filter"]["s_per_step"] * 1e6, 3),
                   "value_without_k1": round(job_ops * args.steps / t_nok1 / 1e12, 3),
                   "note": "the filter transform is offline in the paper (P:370); the headline step includes it"},
            "single_stream": {"ms_per_step": round(single_ms, 5),
                              "tops": round(job_ops / (single_ms / 1e3) / 1e12, 3),
                              "note": "one batch at a time on one stream (latency); the headline runs "
                                      f"{len(lanes)} independent batches on {len(lanes)} streams"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "e2e": e2e,
            "self_check": self_check,
            "scaling_error": scal_err,
            "sharded_check": sharded_check,
        }
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _self_check_layer(args, layer, sh, y_dev, S, u8, zp):
    """One image of the timed graphs' output (this rank's first image, set 0) against the CPU oracle."""
    from oracle import oracle as O
    O.build()
    if args.scaling != "strong":
        return {"note": "replica mode: per-rank seeds, not checked"}
    x, w = synth.config_inputs(args.config)               # set 0: the whole seeded batch (w is drawn after x)
    x1 = np.ascontiguousarray(x[sh["n0"]: sh["n0"] + 1])
    w1 = np.ascontiguousarray(w[sh["co0"]: sh["co0"] + sh["co"]])
    if u8:
        xu, wu = (x1.astype(np.int16) + 128).astype(np.uint8), (w1.astype(np.int16) + 128).astype(np.uint8)
        fn = O.wino2_conv_u8 if args.alg == "f2" else O.wino_conv_u8
        ref = fn(xu, wu, zp, zp, layer.pad, O.NHWC, layer.scaling, target=args.target, M0=1, S=S).y8
    else:
        fn = O.wino2_conv if args.alg == "f2" else O.wino_conv
        ref = fn(x1, w1, layer.pad, O.NHWC, layer.scaling, target=args.target, M0=1, S=S).y8
    got = y_dev[:1].cpu().numpy()
    return {"image": int(sh["n0"]), "equal_to_oracle": bool(np.array_equal(got, ref)),
            "elements": int(ref.size), "reference": "oracle (plain C, the paper's pipeline)"}


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


def run_e2e(conv, xs, ws, S, stream, n_sets, reps, dist, dev, job_ops, empty, n_streams=3):
    """Same metric through the C ABI with HOST buffers: every step copies x and w from pinned host
    memory, runs K1..K4 (wino_transform_filter + wino_conv2d_int8_host, whose H2D / D2H copies are
    inside the call) and reads y back to pinned host memory.  Steps rotate over `n_streams` streams,
    each with its own device buffers, so one step's copies overlap another's compute."""
    import torch
    from paper_1901_01965_b200 import _lib as L
    if empty:                                  # join the collectives of the other ranks
        t = torch.zeros(1, dtype=torch.float64, device=dev)
        if dist is not None:
            dist.barrier()
            dist.barrier()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return None
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
            "xd": torch.empty(conv.x_shape, dtype=xs[0].dtype, device=dev),
            "yd": torch.empty(conv.y_shape, dtype=torch.int8, device=dev),
            "wd": torch.empty(conv.w_shape, dtype=ws[0].dtype, device=dev),
            "ww": torch.empty_like(conv.w_wino), "cd": torch.empty_like(conv.codes),
            "ws": torch.empty_like(conv.workspace),
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
    if dist is not None:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    v = job_ops * reps / float(t.item()) / 1e12
    return {"value": round(v, 3), "unit": "TOPS", "h2d_bytes_per_step": int(info.x_bytes + np.prod(conv.w_shape)),
            "d2h_bytes_per_step": int(info.y_bytes), "steps": reps, "streams": n_streams,
            "ms_per_step": round(float(t.item()) * 1e3 / reps, 4), "host_issue_ms_per_step": round(host_issue * 1e3, 4)}


# ----------------------------------------------------------------------------- GPU arm, VGG-16 stack (C5)
def run_ours_stack(args):
    """--config C5: the VGG-16 13-layer stack (BASELINE configs[4]) per step: 13 filter transforms
    + 13 convs (requantised) + 4 max pools; the batch of 256 partitioned over the ranks."""
    import torch

    from paper_1901_01965_b200 import _lib as L
    from paper_1901_01965_b200.stack import ConvStack

    rank, local_rank, world = _env_rank()
    dist = _init_dist(world, local_rank)
    local_rank = _device_index(local_rank)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synth.CONFIGS["C5"]
    shifts = synth.stack_shifts("C5")
    n_all = cfg.layers[0].n
    sh = _shard(args, n_all, cfg.layers[0].c_out, world, rank)      # batch 256 >= world: by batch
    n = sh["n"]
    path = {"staged": L.WINO_PATH_STAGED, "fused": L.WINO_PATH_FUSED, "auto": L.WINO_PATH_AUTO}[args.path]
    st = ConvStack(n, cfg.layers, cfg.pools_after, shifts, device=local_rank, path=path, workspace_mb=args.chunk_mb,
                   lanes=args.lanes)
    n_sets = 2
    xs, wss = [], []
    for i in range(n_sets):
        if args.scaling == "strong":            # the global batch of set i, this rank's images
            x, ws = synth.stack_inputs("C5", rank=i)
            x = np.ascontiguousarray(x[sh["n0"]: sh["n0"] + n])
        else:
            x, ws = synth.stack_inputs("C5", rank=rank * 1000 + i)
        xs.append(torch.from_numpy(x).to(dev))
        wss.append([torch.from_numpy(w).to(dev) for w in ws])
    stream = torch.cuda.Stream(device=dev)

    def step(j, k1=True):
        if k1:
            st.step(xs[j], wss[j], stream)     # the 13 filter transforms forked onto a side stream
        else:
            st(xs[j], stream)

    graphs, graphs_nok1 = [], []
    with torch.cuda.stream(stream):
        for j in range(n_sets):                 # the code buffers seen once, outside the graphs
            step(j)
        for i in range(args.warmup):
            step(i % n_sets)
        stream.synchronize()
        for j in range(n_sets):
            for k1, gl in ((True, graphs), (False, graphs_nok1)):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    step(j, k1)
                gl.append(g)
        for j in range(3):
            graphs[j % n_sets].replay()
        stream.synchronize()

    def run_steps(k, gl=graphs):
        with torch.cuda.stream(stream):
            for i in range(k):
                gl[i % n_sets].replay()

    ops_local = sum(synth.direct_ops(l, n=n) for l in cfg.layers)
    job_ops = sum(synth.direct_ops(l) for l in cfg.layers) * (world if args.scaling == "weak" else 1)
    with ClockSampler(local_rank) as clk:
        t_max = _timed([stream], lambda: run_steps(args.steps), dist, dev)
    value = job_ops * args.steps / t_max / 1e12
    per_step = t_max / args.steps
    trials = _trials(run_steps, per_step, job_ops, dist, [stream], dev)
    t_nok1 = _timed([stream], lambda: run_steps(args.steps, graphs_nok1), dist, dev)
    # self-check: set 0 through the timed graph, this rank's first image against the oracle stack
    graphs[0].replay()
    stream.synchronize()
    y_first = st.pooled.get(len(cfg.layers) - 1, st.outs[-1])[:1].cpu().numpy()
    peaks = _peaks()
    # per-layer kernels timed alone on the stack's own buffers (outside the timed region)
    kern_l, cur = [], xs[0]
    for i, c in enumerate(st.convs):
        kern_l.append(profile_kernels(c, [cur], [wss[0][i]], [st.outs[i]], shifts[i], stream, 1,
                                      max(10, 2 * c.info.n_chunks), lanes=c.info.lanes))
        cur = st.pooled.get(i, st.outs[i])
    t_roof = 0.0
    for l, c in zip(cfg.layers, st.convs):
        t_roof += conv_roof_s(c.info, l.c_in, l.c_out, peaks)[0]
    dom_l = max(range(len(st.convs)), key=lambda i: max(k["s_per_step"] for k in kern_l[i].values()))
    dk = max(kern_l[dom_l], key=lambda k: kern_l[dom_l][k]["s_per_step"])
    lay, cdom = cfg.layers[dom_l], st.convs[dom_l]
    roof = kernel_roofline(dk, kern_l[dom_l], cdom.info, lay.c_in, lay.c_out, peaks, min(cdom.info.chunk_images, n))
    roof["layer"] = dom_l + 1
    roof["traffic"] = load_traffic(f"C5_L{dom_l + 1}").get(dk)
    roof["peak_source"] = peaks["source"] + (" (int8 = 2 x bf16 burst)" if roof["bound"] == "tensor"
                                             else " (hbm_gbs, burst copy)")
    stack_kernel_us = sum(k["s_per_step"] for kl in kern_l for k in kl.values()) * 1e6
    layers_us = [round(sum(k["s_per_step"] for k in kl.values()) * 1e6, 1) for kl in kern_l]
    layers_roof = [round(kernel_roofline(max(kl, key=lambda k: kl[k]["s_per_step"]), kl, c.info, l.c_in, l.c_out,
                                         peaks, min(c.info.chunk_images, n))["frac"], 4)
                   for kl, c, l in zip(kern_l, st.convs, cfg.layers)]
    k1_us = sum(kl["k1_filter"]["s_per_step"] for kl in kern_l) * 1e6
    # e2e: host x in, host final activation out (pinned), copies inside the region, through the C ABI
    xh = xs[0].cpu().pin_memory()
    out = st(xs[0], stream)
    torch.cuda.synchronize()
    yh = torch.empty(out.shape, dtype=torch.int8).pin_memory()
    xd = torch.empty_like(xs[0])
    reps = 3
    if dist is not None:
        dist.barrier()
    with torch.cuda.stream(stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(reps):
            xd.copy_(xh, non_blocking=True)
            step_out = st.step(xd, wss[0], stream)
            yh.copy_(step_out, non_blocking=True)
        e1.record(stream)
        stream.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    te = float(te.item())
    if rank == 0:
        self_check, oracle_out = _self_check_stack(y_first, sh["n0"], shifts, args.scaling)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 4), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "int8", "data": "synthetic",
            "config": {"workload": f"C5: {cfg.description}", "batch": n_all, "batch_per_gpu": n,
                       "layers": len(cfg.layers), "layout": "NHWC", "filter_scaling": True, "requant_shifts": shifts,
                       "step": "13 filter transforms + 13 convs + 4 max pools",
                       "paths": ["fused" if c.info.path == L.WINO_PATH_FUSED else "staged" for c in st.convs],
                       "l2": "activations 0.8 GB per layer >> 126 MiB L2; 2 input sets rotated",
                       "chunk_mb": args.chunk_mb, "chunks": [c.info.n_chunks for c in st.convs],
                       "lanes": [c.info.lanes for c in st.convs],
                       "parallelism": f"dp{world}: " + ("batch-partitioned (strong scaling)" if args.scaling == "strong"
                                                        else "replicated per-rank batches (weak scaling)") +
                                      "; no data-path collective"},
            "roofline": roof,
            "path_roofline": {"t_roof_us": round(t_roof * 1e6, 2), "t_step_us": round(per_step * 1e6, 2),
                              "frac": round(t_roof / per_step, 4),
                              "roofline_effective_tops": round(ops_local / t_roof / 1e12, 1),
                              "basis": "sum over layers of max(2*46*T*Cin*Cout / int8 burst, (x+y+W') / HBM)"},
            "trials": trials,
            "k1": {"us_per_step": round(k1_us, 1), "value_without_k1": round(job_ops * args.steps / t_nok1 / 1e12, 3),
                   "note": "13 filter transforms, offline in the paper (P:370); the headline step includes them"},
            "kernel_sum_vs_step": round(stack_kernel_us / (per_step * 1e6), 3),
            "layers_kernel_us": layers_us,
            "layers_kernels_us": [{k: round(v["s_per_step"] * 1e6, 1) for k, v in kl.items()} for kl in kern_l],
            "layers_dominant_kernel_frac": layers_roof,
            "gpu_launches": st.launches() * args.steps,   # per layer K1 + K2..K4 per chunk, + the pools
            "clocks": clk.summary(),
            "e2e": {"value": round(job_ops * reps / te / 1e12, 3), "unit": "TOPS",
                    "h2d_bytes_per_step": int(xh.numel()), "d2h_bytes_per_step": int(yh.numel()),
                    "steps": reps},
            "self_check": self_check,
        }
        if not args.no_cpu and world == 1:
            line["cpu_baseline"] = cpu_baseline_stack(shifts, oracle_out)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _oracle_stack_image(img, shifts):
    """One image of the C5 batch through the oracle's 13 layers + pools (plain C): (output, seconds)."""
    from oracle import oracle as O
    O.build()
    cfg = synth.CONFIGS["C5"]
    x, ws = synth.stack_inputs("C5", n=img + 1)
    cur = np.ascontiguousarray(x[img: img + 1])
    t0 = time.perf_counter()
    for i, w in enumerate(ws):
        cur = O.wino_conv(cur, w, 1, O.NHWC, scaling=True, M0=1, S=shifts[i]).y8
        if i in cfg.pools_after:
            cur = O.maxpool2(cur, O.NHWC)
    return cur, time.perf_counter() - t0


def _self_check_stack(y_first, img, shifts, scaling):
    if scaling != "strong":
        return {"note": "replica mode: per-rank seeds, not checked"}, None
    ref, t = _oracle_stack_image(img, shifts)
    return {"image": int(img), "equal_to_oracle": bool(np.array_equal(y_first, ref)), "elements": int(ref.size),
            "reference": "oracle.wino_conv x 13 + maxpool2 (plain C)"}, (ref, t, img)


def cpu_baseline_stack(shifts, oracle_out=None):
    """The oracle as it stands on the host cores: image 0 of C5 through the 13 layers with the
    Winograd pipeline (the same run as the self-check), and the direct convolution (O1) of every layer
    on that image's activations."""
    from oracle import oracle as O
    O.build()
    cfg = synth.CONFIGS["C5"]
    if oracle_out is None or oracle_out[2] != 0:
        _, t = _oracle_stack_image(0, shifts)
    else:
        t = oracle_out[1]
    ops = sum(synth.direct_ops(l, n=1) for l in cfg.layers)
    x, ws = synth.stack_inputs("C5", n=1)
    cur, td = x, 0.0
    for i, w in enumerate(ws):
        t0 = time.perf_counter()
        O.direct_conv(cur, w, 1, O.NHWC)
        td += time.perf_counter() - t0
        cur = O.wino_conv(cur, w, 1, O.NHWC, scaling=True, M0=1, S=shifts[i]).y8
        if i in cfg.pools_after:
            cur = O.maxpool2(cur, O.NHWC)
    cores = len(os.sched_getaffinity(0))
    return {"value": round(ops / t / 1e12, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"oracle.wino_conv x 13 + pools (plain C, OpenMP {cores} threads) on image 0 of C5 "
                      f"({ops:.3e} direct ops); {t:.2f} s",
            "direct": {"value": round(ops / td / 1e12, 6), "unit": "TOPS",
                       "sample": f"oracle.direct_conv (O1) of the 13 layers on image 0; {td:.2f} s"}}


# ----------------------------------------------------------------------------- CPU oracle arm
def _oracle_sample(config, budget_s, layer_index=0):
    """A bounded sample of the workload for the CPU oracle: the first `rows` input rows of one image of
    layer `layer_index` (pad 1), sized to ~budget_s seconds.  Returns (run, rows, direct ops)."""
    from oracle import oracle as O
    cfg = synth.CONFIGS[config]
    layer = cfg.layers[layer_index]
    x, w = synth.config_inputs(config, n=1, layer=layer_index)
    S = synth.requant_shift(layer)

    def run(rows, direct=False):
        xs = np.ascontiguousarray(x[:, :rows])
        t0 = time.perf_counter()
        if direct:
            O.direct_conv(xs, w, layer.pad, O.NHWC)
        else:
            O.wino_conv(xs, w, layer.pad, O.NHWC, scaling=layer.scaling, M0=1, S=S)
        return time.perf_counter() - t0

    rows = min(layer.h, 4)
    dt = run(rows)
    while rows < layer.h and dt < budget_s / 3:
        rows = min(layer.h, rows * 2)
        dt = run(rows)
    ops = synth.direct_ops(synth.LayerCfg(1, rows, layer.w, layer.c_in, layer.c_out, layer.pad))
    return run, rows, ops


def cpu_baseline(config, budget_s=10.0):
    from oracle import oracle as O
    O.build()
    run, rows, ops = _oracle_sample(config, budget_s / 2)
    reps, t = 0, 0.0
    while t < budget_s / 2 or reps < 1:
        t += run(rows); reps += 1
    td, nd = 0.0, 0
    while td < budget_s / 8 or nd < 1:
        td += run(rows, direct=True); nd += 1
    cores = len(os.sched_getaffinity(0))
    return {"value": round(ops * reps / t / 1e12, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"oracle.wino_conv (plain C, OpenMP {cores} threads) on image 0 rows 0..{rows - 1} "
                      f"of {config} ({ops:.3e} direct ops) x {reps}; {t:.2f} s",
            "direct": {"value": round(ops * nd / td / 1e12, 6), "unit": "TOPS",
                       "sample": f"oracle.direct_conv (O1) on the same rows x {nd}; {td:.2f} s"}}


def run_reference(args):
    rank, _, world = _env_rank()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    cfg = synth.CONFIGS[args.config]
    per_step_budget = max(0.05, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    # C5: the steps cycle through the 13 layers (a row stripe of one image each); C1-C4: the one layer
    samples = [_oracle_sample(args.config, per_step_budget, li) for li in range(len(cfg.layers))]
    for i in range(args.warmup):
        run, rows, _ = samples[i % len(samples)]
        run(rows)
    t, ops = 0.0, 0
    for i in range(args.steps):
        run, rows, o = samples[i % len(samples)]
        t += run(rows)
        ops += o
    v = ops / t / 1e12
    cores = len(os.sched_getaffinity(0))
    layer = cfg.layers[0]
    what = ("per step: oracle.wino_conv on a row stripe of image 0 of layer (step mod 13)"
            if len(samples) > 1 else f"per step: oracle.wino_conv on image 0 rows 0..{samples[0][1] - 1}")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "TOPS", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3 / args.steps, 3),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int8",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.description}", "batch": layer.n, "h": layer.h,
                       "w": layer.w, "c_in": layer.c_in, "c_out": layer.c_out, "layout": "NHWC",
                       "filter_scaling": layer.scaling, "layers": len(cfg.layers)},
            "cpu_baseline": {"value": round(v, 6), "unit": "TOPS", "cores": cores, "kind": "oracle",
                             "cpu_model": _cpu_model(), "sample": f"{what} ({ops:.3e} direct ops in total)"},
            "e2e": {"value": round(v, 6), "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default per config: C5 50, C1-C3 2000)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (default): the configuration's batch is partitioned over the ranks (Cout for "
                         "batch 1), as BASELINE north_star says; weak: every rank runs a whole batch")
    ap.add_argument("--streams", type=int, default=3,
                    help="C1-C4: independent batches in flight on separate streams (own filter/workspace buffers)")
    ap.add_argument("--path", default="auto", choices=["auto", "fused", "staged"],
                    help="auto (the plan picks fused for c_in <= 128, staged otherwise)")
    ap.add_argument("--input", default="i8", choices=["i8", "u8"],
                    help="u8: uint8 tensors with zero points (SURVEY f2; either algorithm and path, c_in <= 224)")
    ap.add_argument("--alg", default="f4", choices=["f4", "f2"],
                    help="f4: complex F(4x4,3x3) (the north star); f2: rational F(2x2,3x3) (SURVEY f1, either path)")
    ap.add_argument("--target", type=int, default=255, choices=[255, 127],
                    help="filter scaling target: 255 = the paper's (two-piece W'); 127 = int8-native single-piece "
                         "W' (SURVEY f3, staged F(4x4) int8)")
    ap.add_argument("--e2e-streams", type=int, default=3,
                    help="host-buffer (e2e) leg: steps in flight on separate streams, so copies overlap compute")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=24.0,
                    help="CPU oracle baseline budget (about half of it is the timed sample)")
    ap.add_argument("--chunk-mb", type=int, default=256,
                    help="C5: per-layer batch-chunk budget for the V (+ M'') workspace in MiB (wino_conv_desc.workspace_mb)")
    ap.add_argument("--lanes", type=int, default=3,
                    help="C5: concurrent chunk pipelines inside each conv call (wino_conv_desc.lanes; 0 = one)")
    ap.add_argument("--plan-only", action="store_true", help="CPU/gloo: spawn the ranks and print their shards")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = DEFAULT_STEPS[args.config]
    if args.warmup < 3:
        args.warmup = 3
    _, _, world = _env_rank()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    if world != args.gpus and args.impl == "ours":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
        sys.exit(2)
    if args.plan_only:
        run_plan_only(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.config == "C5":
        if args.alg != "f4" or args.input != "i8" or args.target != 255:
            print("bench.py: C5 runs the north-star variant (F4x4, int8, target 255) only", file=sys.stderr)
            sys.exit(2)
        run_ours_stack(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
