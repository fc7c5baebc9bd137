"""bench.py — train samples/s of the eager training step (fwd + bwd + SGD)
on synthetic data (BASELINE.json metric), one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N      (N > 1: data parallel, NCCL buckets)

Default workload = the north-star configuration (BASELINE.json configs[3],
C4: ResNet-50 v1.5, 224x224, batch 256/GPU, bf16); `--config c1|c2|c3|c5`
selects the others.  Prints ONE JSON line on rank 0.  `--gpus N` without a
torchrun environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1 rendezvous).

`--impl reference` times the float64 CPU oracle (oracle/) on this host — the
reference arm of this tier (no reference implementation exists; see
DESIGN.md).  It is the only other place this file executes oracle/ besides
the cpu_baseline leg.
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

CONFIGS = {
    "c1": dict(workload="C1 MLP 784-128-10, batch 64, fp32 (3xTF32 GEMMs)", net="mlp", sizes=(784, 128, 10),
               batch=64, dtype="f32"),
    "c2": dict(workload="C2 MLP 4096-4096-4096-1000, batch 1024/GPU, bf16", net="mlp",
               sizes=(4096, 4096, 4096, 1000), batch=1024, dtype="bf16"),
    "c3": dict(workload="C3 AlexNet (single tower), 224x224, batch 256/GPU, bf16", net="alexnet", batch=256,
               dtype="bf16"),
    "c4": dict(workload="C4 ResNet-50 v1.5, 224x224, batch 256/GPU, bf16", net="resnet50", batch=256, dtype="bf16"),
    "c6": dict(workload="C6 VGG-19, 224x224, batch 256/GPU, bf16 (Table 1 CNN; dropout 0.5 on fc6/fc7)", net="vgg19",
               batch=256, dtype="bf16"),
    "c7": dict(workload="C7 MobileNetV2, 224x224, batch 256/GPU, bf16 (Table 1 \"MobileNet\"; depthwise convs, "
                        "ReLU6, dropout 0.2)", net="mobilenetv2", batch=256, dtype="bf16"),
    "c5": dict(workload="C5 NCF NeuMF (ML-20M tables), batch 8192/GPU (65536 global on 8), bf16; embedding "
                        "tables on sparse touched-rows SGD", net="ncf", batch=8192, dtype="bf16", sparse=True),
}
METRIC = "train samples/s (fwd+bwd+SGD) at 1/2/4/8 B200; per-kernel % of roofline"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ---------------------------------------------------------------- synthetic workloads
def make_model(cfg, be, seed=0):
    import synth
    if cfg["net"] == "mlp":
        m = be.nn.MLP(cfg["sizes"])
    elif cfg["net"] == "alexnet":
        m = be.nn.AlexNet()
    elif cfg["net"] == "resnet50":
        m = be.nn.ResNet50(bn_stats=os.environ.get("BENCH_BN_STATS", "1") == "1")
    elif cfg["net"] == "vgg19":
        m = be.nn.VGG19()
    elif cfg["net"] == "mobilenetv2":
        m = be.nn.MobileNetV2()
    else:
        m = be.nn.NCF()
    m.load(synth.make_params(m.param_specs(), seed))
    return m


def host_batch(cfg, seed, rank=0):
    """Host arrays of one batch in the device layout (marshalling only)."""
    import synth
    B = cfg["batch"]
    from paper_1912_01703_b200.api import f32_to_bf16_bits
    if cfg["net"] == "mlp":
        x = (synth.uniform if cfg["sizes"][0] == 784 else synth.normal)((B, cfg["sizes"][0]), seed, 1 + rank)
        y = synth.labels(B, cfg["sizes"][-1], seed + rank)
        xd = f32_to_bf16_bits(x) if cfg["dtype"] == "bf16" else x
        return [xd, y]
    if cfg["net"] in ("alexnet", "resnet50", "vgg19", "mobilenetv2"):
        x = synth.normal((B, 3, 224, 224), seed, 1 + rank)
        nhwc = np.zeros((B, 224, 224, 8), np.float32)
        nhwc[..., :3] = x.transpose(0, 2, 3, 1)
        y = synth.labels(B, 1000, seed + rank)
        return [f32_to_bf16_bits(nhwc) if cfg["dtype"] == "bf16" else nhwc, y]
    u, i, y = synth.ncf_batch(B, 138493, 26744, seed + rank)
    return [u, i, y]


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every 10 ms while the
    timed region runs (the recipe's clocks line; nvidia-smi -lms cannot
    sample a few-ms region)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index, self.samples, self.stop_flag = index, [], False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.01)

    def stop(self):
        self.stop_flag = True
        if getattr(self, "nv", None) is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        self.thread.join(timeout=1)
        sm = [s for s, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(sm), "source": "nvml 10 ms"}


# ---------------------------------------------------------------- oracle timing (reference arm / cpu_baseline)
def oracle_time(cfg, budget_s=15.0, max_steps=None, min_steps=1):
    """Time the float64 oracle's train_step on a bounded sample of the workload."""
    import synth
    from oracle import nets as onets
    from oracle.step import train_step
    B = cfg["batch"]
    if cfg["net"] == "mlp":
        net = onets.MLP(cfg["sizes"])
        sb = min(B, 256 if cfg["sizes"][0] > 1000 else B)
        batch = ((synth.uniform if cfg["sizes"][0] == 784 else synth.normal)((sb, cfg["sizes"][0]), 0, 1),
                 synth.labels(sb, cfg["sizes"][-1], 0))
    elif cfg["net"] in ("alexnet", "resnet50", "vgg19", "mobilenetv2"):
        net = {"alexnet": onets.AlexNet, "resnet50": onets.ResNet50, "vgg19": onets.VGG19,
               "mobilenetv2": onets.MobileNetV2}[cfg["net"]]()
        sb = 2
        batch = (synth.normal((sb, 3, 224, 224), 0, 1), synth.labels(sb, 1000, 0))
    else:
        net = onets.NCF()
        sb = 8192
        batch = synth.ncf_batch(sb, 138493, 26744, 0)
    P = synth.make_params(net.param_specs(), 0)
    t0 = time.perf_counter()
    n = 0
    while True:
        out = train_step(net, P, batch, lr=0.01)
        P = {k: v.astype(np.float32) for k, v in out["params"].items()}
        n += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and n >= min_steps) or (max_steps and n >= max_steps):
            break
    host_cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    threads = blas_threads() or host_cores
    return {"value": n * sb / el, "unit": "samples/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "threads": threads, "host_cores": host_cores,
            "sample": f"{n} float64 oracle step(s) of {cfg['net']} at batch {sb} (of {B}) in {el:.1f}s, "
                      f"NumPy/OpenBLAS on all host cores"}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def blas_threads():
    """Threads the oracle's BLAS actually runs with (threadpoolctl), else the env setting."""
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads") for d in threadpool_info() if d.get("user_api") == "blas"]
        if n:
            return max(n)
    except Exception:
        pass
    return int(os.environ.get("OPENBLAS_NUM_THREADS", "0")) or None


# ---------------------------------------------------------------- our arm
def run_ours(args, cfg, rank, world, local_rank):
    import torch
    import paper_1912_01703_b200 as be
    torch.cuda.set_device(local_rank)
    stream = torch.cuda.Stream(priority=-1)  # compute stream outranks the side streams
    be.init(local_rank, stream.cuda_stream)
    be.set_compute_dtype(cfg["dtype"])
    dist = None
    if world > 1:
        import torch.distributed as dist
        uid = [be.dist_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        be.dist_init(rank, world, uid[0])
    model = make_model(cfg, be, seed=0)
    params = model.parameters()
    dp_mode = None
    if world > 1:
        # embedding tables on the sparse path exchange lookups, not gradients
        tables = model.embedding_tables() if cfg.get("sparse") else []
        dp_params = [p for p in params if all(p is not t for t in tables)]
        if args.dp == "p2p":
            # fused allreduce + SGD over CUDA-IPC peer memory (be_p2p_*);
            # every rank built identical parameters from the same seed
            blob = be.p2p_attach(dp_params, rank, world, 25 << 20)
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
            be.p2p_connect(blobs)
        else:
            be.ddp_attach(dp_params, 25 << 20)
        dp_mode = args.dp
    hb = host_batch(cfg, seed=1, rank=rank)
    dts = ["bf16" if (i == 0 and cfg["net"] not in ("ncf",) and cfg["dtype"] == "bf16") else None
           for i in range(len(hb))]

    def dev_batch():
        out = []
        for a, d in zip(hb, dts):
            if d == "bf16":
                t = be.empty(a.shape, "bf16")
                be.api.call("be_tensor_copy_from_host_async", t.handle, a.ctypes.data_as(__import__("ctypes").c_void_p),
                            a.nbytes)
                out.append(t)
            else:
                out.append(be.tensor(a))
        be.synchronize()
        return out
    batch = dev_batch()

    def step(b, overlap=args.sgd == "overlap"):
        return be.nn.train_step(model, b, lr=0.01, momentum=0.9, weight_decay=1e-4, overlap_sgd=overlap,
                                sparse_embeddings=cfg.get("sparse", False))

    # setup: on-line kernel-variant autotuning (each tuned shape runs every
    # candidate twice, cudnn.benchmark-style) before the W warm-up steps
    # (in the timed mode, so the fused-SGD GEMM variants are tuned too; the
    # side-stream update then only carries the small bias/BN parameters)
    for _ in range(args.tune_steps):
        step(batch)
    # host cost of the eager step itself: one step enqueued onto an idle GPU
    # (empty launch queue).  In the back-to-back loops the host blocks inside
    # the driver once the launch queue is full, so their host time tracks the
    # GPU time rather than the enqueue cost (Fig. 1).
    idle = []
    for _ in range(5):
        be.synchronize()
        ta = time.perf_counter()
        step(batch)
        idle.append((time.perf_counter() - ta) * 1e3)
    be.synchronize()
    host_idle_ms = statistics.median(idle)
    loss = None
    for _ in range(args.warmup):
        loss = step(batch)  # held like the timed loop does (the previous loss stays alive one step)
    be.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        be.synchronize()
    # the clock sampler (NVML init + its thread) starts before the settle steps,
    # so its start-up latency does not leave the GPU idle (clocks dropping) right
    # before the timed region — which made the first pass of the launch-bound
    # configs (C1, C5) run below the later passes; its samples are cleared at
    # the start of the timed region
    clocks = ClockSampler(local_rank)
    clocks.start()
    # settle: the allocator's pools reach their steady state when a step that
    # starts from a synchronised GPU (as the timed region does) makes no new
    # cudaMalloc; at most 10 such extra warm-up steps
    settle = 0
    for settle in range(1, 11):
        barrier()
        a0 = be.alloc_stats()["raw_alloc_count"]
        loss = step(batch)
        loss = step(batch)
        be.synchronize()
        if be.alloc_stats()["raw_alloc_count"] == a0:
            break
    # steady clocks: the launch-bound configs (C1, C5: 0.2–0.3 ms steps) ramp
    # for tens of ms after the idle gaps above (their passes sped up pass after
    # pass) — extra untimed steps until ≥ 0.25 s of back-to-back stepping
    t_ramp = time.perf_counter()
    ramp = 0
    while time.perf_counter() - t_ramp < 0.25 and ramp < 2000:
        loss = step(batch)
        ramp += 1
        if ramp % 16 == 0:
            be.synchronize()
    be.synchronize()
    stats_warm = be.alloc_stats()
    trace = bool(os.environ.get("BE_ALLOC_TRACE"))

    # ---- device-resident timed region
    if trace:
        print("=== timed region start", file=sys.stderr, flush=True)
    barrier()
    clocks.samples.clear()
    l0 = be.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ selects these launches
    for _ in range(args.steps):
        loss = step(batch)
    torch.cuda.nvtx.range_pop()
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    launches = be.launch_count() - l0
    stats_timed = be.alloc_stats()
    if trace:
        print("=== timed region end", file=sys.stderr, flush=True)
    # further timed passes of the same K steps (the paper's mean ± sd convention,
    # PAPER.md:271-276); the headline value is the first pass
    rep_ms = [ms]
    for _ in range(max(args.repeats, 1) - 1):
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        r0.record(stream)
        for _ in range(args.steps):
            loss = step(batch)
        r1.record(stream)
        barrier()
        rep_ms.append(r0.elapsed_time(r1))
    # second, profiled pass of the same K steps: every tcgen05 GEMM / conv launch
    # bracketed by CUDA events on its stream (the brackets cost a little, so the
    # headline value comes from the unprofiled pass above)
    be.prof_enable(True)
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record(stream)
    for _ in range(args.steps):
        loss = step(batch)
    e5.record(stream)
    barrier()
    be.prof_enable(False)
    ms_prof = e4.elapsed_time(e5)
    prof = be.prof_read()
    clk = clocks.stop()
    stats_after = be.alloc_stats()
    nccl_info = None
    if world > 1:
        t = torch.tensor(rep_ms, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rep_ms = [float(v) for v in t.tolist()]
        ms = rep_ms[0]
        r_, nr = be.api.dist_world()
        nccl_info = {"nranks": nr, "backend": "libbe NCCL communicator (ncclCommCount)",
                     "allreduce": ("fused peer-memory allreduce + SGD kernel per 25 MB bucket (be_p2p_*, CUDA IPC "
                                   "over NVLink), p2p_status=%d" % be.api.p2p_status()) if dp_mode == "p2p" else
                     "bucketed ncclAllReduce(avg), 25 MB fp32 buckets, comm stream"}

    # ---- end-to-end through the public API: every step's batch goes pinned host → device
    # (double-buffered on a copy stream so batch i+1 transfers while step i computes, the
    # data loader's pinned-memory path) and the loss comes back device → host
    # CNN images travel as the real 3 channels (bf16 NHWC, 2.7x fewer bytes over
    # the host link); the device pads them to the kernels' 8-channel layout
    # (concat with a resident zero block) inside the timed step
    hb_e2e, dts_e2e, pad = list(hb), list(dts), None
    if cfg["net"] in ("alexnet", "resnet50", "vgg19", "mobilenetv2") and cfg["dtype"] == "bf16":
        img = hb[0]
        npix = img.shape[0] * img.shape[1] * img.shape[2]
        hb_e2e[0] = np.ascontiguousarray(img[..., :3]).reshape(npix, 3)
        zeros5 = be.tensor(np.zeros((npix, 5), np.float32), dtype="bf16")
        pad = (zeros5, tuple(img.shape))
    pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in hb_e2e]
    loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
    shapes = [(a.shape, d or {np.dtype(np.int32): "i32", np.dtype(np.float32): "f32"}[a.dtype])
              for a, d in zip(hb_e2e, dts_e2e)]
    pipe = be.api.InputPipeline(shapes)
    host = [(p.data_ptr(), p.numel() * p.element_size()) for p in pinned]
    import ctypes as C
    h2d = sum(a.nbytes for a in hb_e2e)

    def e2e_batch(b):
        if pad is None:
            return b
        x8 = be.reshape(be.concat([b[0], pad[0]]), pad[1])
        return [x8] + list(b[1:])

    def e2e_loop(n):
        pipe.put(0, host)
        loss = None
        for i in range(n):
            cur = i % 2
            loss = step(e2e_batch(pipe.get(cur)))
            pipe.release(cur)
            if i + 1 < n:
                pipe.put(1 - cur, host)
            be.api.call("be_tensor_copy_to_host_async", loss.handle, C.c_void_p(loss_host.data_ptr()), 4)
        return loss
    # warm the copy stream / pipeline like the device loop; the host link needs
    # tens of ms of traffic after the device-only passes before it copies at
    # full rate (measured: first 30-step pass 0.58 ms/step, then 0.46-0.47)
    tw = time.perf_counter()
    while True:
        e2e_loop(max(args.warmup, 3))
        barrier()
        if time.perf_counter() - tw > 0.1:
            break
    if os.environ.get("BENCH_E2E_DEBUG"):
        for rep in range(3):
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            e2e_loop(args.steps)
            d1.record(stream)
            barrier()
            print(f"e2e rep {rep}: {d0.elapsed_time(d1) / args.steps:.4f} ms/step", file=sys.stderr, flush=True)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    th0 = time.perf_counter()
    e2e_loop(args.steps)
    host_ms_e2e = (time.perf_counter() - th0) * 1e3 / args.steps
    e3.record(stream)
    barrier()
    ms_e2e = e2.elapsed_time(e3)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    final_loss = float(loss_host.item())

    if rank != 0:
        return None
    B = cfg["batch"]
    value = B * world * args.steps / (ms / 1e3)
    # roofline of the dominant kernel class (tcgen05 GEMM)
    pk, pk_kind = peaks()
    tc = [r for r in prof if r["name"].startswith(("gemm_tc", "conv_tc"))]
    upd = [r for r in prof if r["name"].startswith("gemm_upd")]
    gemm_ms = sum(r["ms"] for r in tc)
    flops = sum(r["flops"] for r in tc)
    achieved = flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else 0.0
    # burst peak (a kernel timed alone at full clock) unless the clocks record of
    # this region shows the power cap / a clock well below max, then sustained
    capped = ("sw_power_cap" in clk["reasons"]) or (clk["sm_mhz"] and clk["sm_max_mhz"]
                                                     and clk["sm_mhz"] < 0.93 * clk["sm_max_mhz"])
    peak_key = "bf16_tflops_sustained" if capped else "bf16_tflops"
    peak = pk.get(peak_key, pk.get("bf16_tflops"))
    dt_bench = "bf16" if cfg["dtype"] == "bf16" else "f32"
    if cfg["dtype"] == "f32":
        peak = peak / 2.0 / 3.0  # tf32 nominal = bf16/2; 3xTF32 issues 3 MMAs per algorithmic product
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4) if peak else None, "traffic": None,
            "kernel": "tcgen05 GEMM + implicit-GEMM conv launches of the step (gemm_tc*, conv_tc*)",
            "launches_per_step": len(tc) / args.steps,
            "share_of_step": round(gemm_ms / ms_prof, 4) if ms_prof else None,
            "profiled_pass_ms_per_step": round(ms_prof / args.steps, 4),
            "peak_source": f"MEASURED_PEAKS.json {peak_key} ({pk_kind}; "
                           + ("power cap / low clock seen in the region)" if capped else "no power cap in the region)")}
    shapes = {}
    for r in tc:
        key = f"{r['m']}x{r['n']}x{r['k']}"
        s = shapes.setdefault(key, [0, 0.0, r["flops"]])
        s[0] += 1
        s[1] += r["ms"]
    roof["per_shape"] = {k: {"launches": v[0], "avg_us": round(v[1] / v[0] * 1e3, 2),
                             "tflops": round(v[2] / (v[1] / v[0] / 1e3) / 1e12, 1)} for k, v in shapes.items()}
    # SURVEY §8(d)'s per-kernel roofline: each launch's ideal time is
    # max(flops / tensor peak, algorithmic bytes / HBM peak); the class figure
    # is Σ ideal / Σ measured (memory-bound shapes — K = 64 1×1 convs, the
    # fused-SGD wgrads — are held to the HBM roof instead of the tensor roof)
    hbm = pk.get("hbm_gbs", 6650.0) * 1e9
    ideal = sum(max(r["flops"] / (peak * 1e12), r["bytes"] / hbm) for r in tc)
    roof["frac_per_kernel_roofline"] = round(ideal / (gemm_ms / 1e3), 4) if gemm_ms else None
    roof["hbm_peak_gbs"] = pk.get("hbm_gbs")
    if upd:
        # wgrad GEMMs carrying the SGD update in their epilogue (be_sgd_overlap):
        # bound by the P/V/shadow traffic (18 B/param) + operand stream
        ums = sum(r["ms"] for r in upd)
        ub = sum(r["bytes"] for r in upd)
        roof["fused_sgd_gemm"] = {"launches_per_step": len(upd) / args.steps, "ms_per_step": round(ums / args.steps, 4),
                                  "achieved_gbs": round(ub / (ums / 1e3) / 1e9, 1), "peak_gbs": pk.get("hbm_gbs"),
                                  "frac": round(ub / (ums / 1e3) / hbm, 4),
                                  "tflops": round(sum(r["flops"] for r in upd) / (ums / 1e3) / 1e12, 1)}
    # traffic: DRAM bytes per launch of this class, from one ncu capture of this
    # config's step (tools/ncu_class.py writes profiles/traffic_<config>.json);
    # used only if that capture is of the same kernel class, else null
    trafficf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(trafficf):
        tj = json.load(open(trafficf))
        if tj.get("kernel_class") == "gemm_tc*,conv_tc*":
            roof["traffic"] = tj.get("dram_bytes_per_launch")
            roof["traffic_source"] = tj.get("source")
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = oracle_time(cfg, budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": dt_bench, "data": "synthetic (seeded, device-resident)",
        "config": {"workload": cfg["workload"], "global_batch": B * world, "per_gpu_batch": B,
                   "parallelism": f"dp{world}", "l2": "working set > L2 (params+grads+momentum stream through "
                   "every step)", "optimizer": "SGD momentum 0.9 wd 1e-4, "
                   + ("overlapped with backward (be_sgd_overlap)" if args.sgd == "overlap" else "fused after backward")
                   + ("; embedding tables: plain SGD on the touched rows inside backward (be_sgd_sparse)"
                      if cfg.get("sparse") else ""),
                   "autotune_steps": args.tune_steps},
        "e2e": {"value": round(B * world * args.steps / (ms_e2e / 1e3), 2), "unit": "samples/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4,
                "host_loop_ms_per_step": round(host_ms_e2e, 4),
                "host_enqueue_ms_per_step": round(host_idle_ms, 4),
                "host_enqueue_note": "host time to enqueue one step onto an idle GPU (median of 5); the e2e loop's "
                                     "host time (host_loop_ms_per_step) includes blocking on the full launch queue"},
        "repeats": {"n": len(rep_ms), "steps_each": args.steps,
                    "samples_per_s": [round(B * world * args.steps / (m / 1e3), 1) for m in rep_ms],
                    "mean": round(statistics.mean(B * world * args.steps / (m / 1e3) for m in rep_ms), 1),
                    "sd": round(statistics.pstdev(B * world * args.steps / (m / 1e3) for m in rep_ms), 1)},
        "nccl": nccl_info,
        "gpu_launches": int(launches),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
        "alloc": {"settle_steps": settle, "clock_ramp_steps": ramp,
                  "raw_alloc_count_delta_timed": stats_timed["raw_alloc_count"] - stats_warm["raw_alloc_count"],
                  "raw_alloc_count_delta_all_passes": stats_after["raw_alloc_count"] - stats_warm["raw_alloc_count"],
                  "peak_bytes_in_use": stats_after["peak_bytes_in_use"]},
        "final_loss": final_loss,
    }
    return line


def run_reference(args, cfg):
    """Reference arm: the float64 oracle on this host's cores, K steps on a
    bounded sample of the workload (each step one oracle train_step)."""
    import synth  # noqa: F401
    t0 = time.perf_counter()
    r = oracle_time(cfg, budget_s=0.0, max_steps=args.warmup, min_steps=1) if args.warmup else None  # warm-up
    r = oracle_time(cfg, budget_s=0.0, max_steps=args.steps, min_steps=args.steps)
    el = time.perf_counter() - t0
    line = {"impl": "reference", "metric": METRIC, "value": round(r["value"], 4), "unit": "samples/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
            "config": {"workload": cfg["workload"], "global_batch": cfg["batch"], "parallelism": "host cores"},
            "cpu_baseline": {"value": round(r["value"], 4), "unit": "samples/s", "cores": r["cores"],
                             "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": round(r["value"], 4), "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": round(el, 1)}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--tune-steps", type=int, default=24, help="untimed autotuning steps before warm-up")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--repeats", type=int, default=5, help="timed passes of K steps (mean ± sd reported)")
    ap.add_argument("--dp", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: p2p = fused allreduce+SGD over peer memory; nccl = bucketed ncclAllReduce")
    ap.add_argument("--sgd", default="overlap", choices=["overlap", "fused"],
                    help="overlap: per-parameter SGD inside backward on a side stream; fused: one launch after")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's own launch form)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, cfg)), flush=True)
        return
    if world > 1:
        # the communicator's init line (nranks, NVLS) goes to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    line = run_ours(args, cfg, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
