#!/usr/bin/env python
"""Benchmark: training images/sec (forward + backward + SGD update) of the
VCNN Imp-6 path on B200, BASELINE.json configs[1] (CIFAR-10-shape 3-conv CNN,
batch 128 per GPU, data-parallel over N GPUs, weak scaling).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One JSON line on rank 0 (driver contract).  `value` is device-timed with CUDA
events per step (each step reads a different batch from a device pool larger
than L2), max over ranks; `e2e` is the same
metric through the C-ABI host entry point (pinned host batch -> H2D -> step ->
D2H loss every step); `roofline` is the dominant kernel's achieved rate over
the timed breakdown pass; `cpu_baseline` is the reference compiled from its
own sources (oracle/_ref), timed on this host.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train images/sec (fwd+bwd+update)"
POOL_BYTES = 256 << 20  # input pool > 126 MB L2: every step's batch comes from HBM


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cifar3")
    ap.add_argument("--batch", type=int, default=128, help="per-GPU batch")
    ap.add_argument("--channels", type=int, default=64, help="single-conv: C_in = C_out")
    ap.add_argument("--ksize", type=int, default=5, help="single-conv: kernel size")
    ap.add_argument("--precision", default="tf32", choices=["tf32", "tf32x3", "fp32"])
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--momentum", type=float, default=0.9)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-infer", action="store_true", help="skip the forward-only pass")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--details", default="", help="write per-op timing JSON here")
    ap.add_argument("--no-roofline-run", action="store_true",
                    help="skip the CIFAR-3 b=1024 conv-GEMM roofline pass")
    ap.add_argument("--no-faithful", action="store_true", help="skip the 3xTF32 pass")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ----------------------------------------------------------------------------
# algorithmic work per op: FLOPs = 2*M*N*K per GEMM, bytes =
# minimal HBM traffic (read inputs once, write outputs once)
# ----------------------------------------------------------------------------
def op_work(spec, B):
    from paper_1501_07338_b200 import spec as S
    chain = spec.chain()
    work = {}
    h, w, c = spec.input
    for i, L in enumerate(spec.layers):
        oh, ow, oc = chain[i]
        nin, nout = B * h * w * c, B * oh * ow * oc
        if isinstance(L, S.ConvSpec):
            kd = c * L.kh * L.kw
            f = 2.0 * B * oh * ow * L.maps * kd
            pw = L.maps * kd + L.maps
            work[(i, "fwd")] = (f, 4.0 * (nin + pw + nout))
            work[(i, "wgrad")] = (f, 4.0 * (nin + nout + pw))
            work[(i, "dgrad")] = (f, 4.0 * (nout + pw + 2 * nin))
        elif isinstance(L, S.PoolSpec):
            work[(i, "fwd")] = (0.0, 4.0 * (nin + 2 * nout))
            work[(i, "dgrad")] = (0.0, 4.0 * (2 * nout + 2 * nin))
            work[(i, "wgrad")] = (0.0, 4.0 * nout)
        else:
            f = 2.0 * B * (h * w * c) * L.units
            pw = L.units * h * w * c + L.units
            work[(i, "fwd")] = (f, 4.0 * (nin + pw + nout))
            work[(i, "wgrad")] = (f, 4.0 * (nin + nout + pw))
            work[(i, "dgrad")] = (f, 4.0 * (nout + pw + 2 * nin))
        h, w, c = oh, ow, oc
    units = spec.output_units()
    work[(len(spec.layers) - 1, "loss")] = (0.0, 4.0 * (2 * B * units + B))
    return work


def op_timing(net, spec, B, steps, load, lr, mom, pk):
    """Eager steps with CUDA events around every op (breakdown mode): rows
    per (layer, op) with algorithmic work and rates, sorted by share."""
    from paper_1501_07338_b200 import spec as S
    net.enable_graph(False)
    net.enable_breakdown(True)
    for i in range(3):  # untimed: first launches of this path's kernels (lazy loading)
        load(i)
        net.train_step(B, lr, mom)
    net.enable_breakdown(True)  # (re-enabling resets the accumulators)
    for i in range(steps):
        load(i)
        net.train_step(B, lr, mom)
    ops = net.read_op_timing()
    bd = net.read_breakdown()
    net.enable_breakdown(False)
    work = op_work(spec, B)
    # the fused tail kernel (launch_mlp_head / launch_head) is timed as the
    # loss op: give it the work of every conv / full layer above the last
    # separately timed one (their forward, both gradients and the loss)
    timed = [l for (l, o) in ops if o != "loss" and l >= 0]
    last = max(timed) if timed else -1
    nl = len(spec.layers)
    tail = [i for i in range(last + 1, nl) if not isinstance(spec.layers[i], S.PoolSpec)]
    tail_name = None
    if (nl - 1, "loss") in ops and tail:
        f = sum(work.get((i, o), (0.0, 0.0))[0] for i in tail for o in ("fwd", "wgrad", "dgrad"))
        by = sum(work.get((i, o), (0.0, 0.0))[1] for i in tail for o in ("fwd", "wgrad", "dgrad"))
        lf, lb = work[(nl - 1, "loss")]
        work[(nl - 1, "loss")] = (f + lf, by + lb)
        tail_name = f"tail(layers {tail[0]}-{tail[-1]} fwd+bwd+loss, one kernel)"
    rows = []
    tot = sum(s for s, _ in ops.values())
    for (layer, op), (sec, cnt) in ops.items():
        f, by = work.get((layer, op), (0.0, 0.0))
        t = sec / cnt
        t_tc = f / (pk["tf32_tflops"] * 1e12) if f else 0.0
        t_hbm = by / (pk["hbm_gbs"] * 1e9) if by else 0.0
        bound = "tensor" if t_tc >= t_hbm else "hbm"
        rows.append({"layer": layer, "op": op, "us": t * 1e6, "share": sec / tot,
                     "flops": f, "bytes": by, "bound": bound,
                     "tflops": f / t / 1e12 if f else 0.0, "gbs": by / t / 1e9 if by else 0.0,
                     "roof_us": max(t_tc, t_hbm) * 1e6})
    rows.sort(key=lambda r: -r["share"])
    return rows, bd, tail_name, tot


def conv_gemm_rows(rows, spec, pk):
    """Per conv GEMM (separately timed fwd / wgrad / dgrad of a conv layer):
    achieved TFLOP/s vs the TF32 peak and vs its own roofline
    min(P_tf32, AI * BW_HBM) with AI from the minimal algorithmic bytes."""
    from paper_1501_07338_b200 import spec as S
    out = []
    for r in rows:
        if r["layer"] < 0 or r["op"] not in ("fwd", "wgrad", "dgrad") or not r["flops"]:
            continue
        if not isinstance(spec.layers[r["layer"]], S.ConvSpec):
            continue
        roof = min(pk["tf32_tflops"], r["flops"] / r["bytes"] * pk["hbm_gbs"] * 1e9 / 1e12)
        out.append({"gemm": f"layer{r['layer']}.{r['op']}", "us": round(r["us"], 2),
                    "tflops": round(r["tflops"], 2),
                    "frac_of_peak": round(r["tflops"] / pk["tf32_tflops"], 4),
                    "roof_tflops": round(roof, 1), "frac_of_roof": round(r["tflops"] / roof, 4),
                    "bound": r["bound"]})
    return sorted(out, key=lambda g: g["gemm"])


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=m["hbm_gbs"], bf16_tflops=m["bf16_tflops"], src="measured")
    except Exception:
        pass
    tf = os.path.join(ROOT, "profiles", "tf32_peak.json")
    if os.path.exists(tf):
        with open(tf) as f:
            p["tf32_tflops"] = json.load(f)["tf32_tflops"]
        p["tf32_src"] = "measured cuBLAS TF32 8192^3 (profiles/tf32_peak.json)"
    else:
        p["tf32_tflops"] = p["bf16_tflops"] / 2
        p["tf32_src"] = "bf16 measured / 2 (dense TF32:BF16 rate ratio)"
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (NVML)."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
                 0x2: "applications_clocks_setting"}
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit and nm != "gpu_idle":
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.nv:
            self.t.join()

    def result(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------
# the reference arm / CPU baseline: the reference's own Executor<float>(imp6)
# run_batch + sgd_step, compiled from its sources (oracle/_ref)
# ----------------------------------------------------------------------------
def cpu_reference(spec, B, steps, warmup, seconds=None):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ctypes as C

    import oracle_py as O
    R = O.ref()
    kind = "reference"
    if R is None:
        return None
    cores = R.ref_max_threads()
    net = O.make_net(spec)
    h = R.ref_bench_create(C.byref(net), B, 8, 0.01, 0.9)
    for _ in range(warmup):
        R.ref_bench_step(h, 1)
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        R.ref_bench_step(h, 1)
        times.append(time.perf_counter() - t0)
        if seconds is None and len(times) >= steps:
            break
        if seconds is not None and (time.perf_counter() - t_start >= seconds and len(times) >= 3):
            break
    R.ref_bench_destroy(h)
    total = sum(times)
    return {"value": B * len(times) / total, "unit": "img/s", "cores": cores, "kind": kind,
            "sample": f"{len(times)} steps of batch {B} ({os.path.basename(O.ref_path())}, "
                      f"Executor<float>(imp6).run_batch + sgd_step, OpenMP {cores} threads)",
            "ms_per_step": 1e3 * total / len(times), "cpu_model": cpu_model()}


def make_spec(args):
    from paper_1501_07338_b200 import spec as S
    if args.config == "single-conv":
        return S.single_conv(channels=args.channels, k=args.ksize)
    return S.PRESETS[args.config]()


def cpu_model():
    """`lscpu` model name of this host."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def bench_config(args, world):
    """The workload description both arms print (identical dicts)."""
    return {"workload": workload_name(args), "per_gpu_batch": args.batch,
            "global_batch": args.batch * world, "parallelism": f"dp{world}",
            "l2": "inputs > L2: distinct batches cycled from a 256 MiB device pool, staged "
                  "by a kernel inside each timed step (GPU arm)",
            "update": f"sgd momentum {args.momentum} lr {args.lr}"}


def workload_name(args):
    if args.config == "single-conv":
        return f"single-conv-c{args.channels}-k{args.ksize}-b{args.batch}-train"
    return f"{args.config}-b{args.batch}-train"


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1501_07338_b200 import spec as S
    spec = make_spec(args)
    r = cpu_reference(spec, args.batch, args.steps, args.warmup)
    if r is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return
    line = {"metric": METRIC, "value": r["value"], "unit": "img/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Rng(8) stream, bench.cpp:29-45)",
            "config": bench_config(args, world),
            "impl": "reference", "where": "host CPU, rank 0 only",
            "cpu_baseline": {"value": r["value"], "unit": "img/s", "cores": r["cores"],
                             "kind": "reference", "sample": r["sample"],
                             "cpu_model": r["cpu_model"]},
            "e2e": {"value": r["value"], "unit": "img/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1501_07338_b200 import _lib, spec as S
    from paper_1501_07338_b200.engine import Network

    rank, world, local = dist_env()
    assert world == args.gpus or world == 1, "launch N>1 under torchrun"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    spec = make_spec(args)
    B = args.batch
    prec = S.Precision[args.precision]
    lr, mom = args.lr, args.momentum

    # synthetic data: the global batch from one Rng(8) stream, sharded contiguously
    xg, clsg, valsg = S.synth_bench_data(spec, B * world, 8)
    sl = slice(rank * B, (rank + 1) * B)
    x_host = torch.from_numpy(np.ascontiguousarray(xg[sl]).reshape(B, -1)).pin_memory()
    is_ce = spec.loss == S.LossKind.softmax_ce
    t_host = torch.from_numpy(np.ascontiguousarray(clsg[sl] if is_ce else valsg[sl])).pin_memory()

    stream = torch.cuda.current_stream()
    net = Network(spec, B, prec, stream=stream)
    net.load_batch(x_host.to(dev), cls=t_host.to(dev) if is_ce else None,
                   values=None if is_ce else t_host.to(dev))
    params, grads, _ = net.device_tensors()
    # device input pool larger than L2, cycled one batch per step (the D2D
    # staging copy into the net's input slot is inside the timed step)
    nbatch = max(2, -(-POOL_BYTES // (x_host.numel() * 4)))
    xp, cp, vp = S.synth_bench_data(spec, B * nbatch, 9 + rank)
    pool_x = torch.from_numpy(xp.reshape(nbatch, B, -1)).to(dev)
    pool_t = torch.from_numpy((cp.reshape(nbatch, B) if is_ce else vp.reshape(nbatch, B, -1))).to(dev)
    del xp, cp, vp

    # the pool as the net's device batch ring: every training step stages its
    # next batch with a kernel inside the step's graph (vcnn_net_set_batch_ring)
    net.set_batch_ring(pool_x, pool_t)

    def load(i):
        pass  # (the ring stages inside the step)

    def load_copy(i):  # forward-only / eager passes: stage explicitly
        j = i % nbatch
        if is_ce:
            net.load_batch(pool_x[j], cls=pool_t[j])
        else:
            net.load_batch(pool_x[j], values=pool_t[j])

    # ---- the step ----
    exchange = None
    if world == 1:
        net.enable_graph(not args.no_graph)

        def step():
            net.train_step(B, lr, mom)
    else:
        # data parallel through the C ABI (vcnn_dp_init: NCCL bootstrap, IPC
        # peer mappings): the graph-replayed step is run_batch(shard) -> ONE
        # kernel reading every replica's gradient over NVLink (rank-ordered
        # weighted sum) + SGD + weight packs; NCCL all-reduce if no P2P path
        from paper_1501_07338_b200.dp import NCCL, P2P, DataParallel
        dp = DataParallel(net)
        net.enable_graph(not args.no_graph)

        def step():
            dp.train_step(B, lr, mom)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        load(i)
        step()
    barrier()
    if world > 1:
        # a P2P exchange whose barrier timed out on any rank -> every rank
        # switches to the NCCL exchange (and says so)
        ok = 1.0
        try:
            dp.status()
        except Exception as e:  # noqa: BLE001
            print(f"[rank {rank}] P2P exchange failed ({e}); NCCL fallback", file=sys.stderr)
            ok = 0.0
        t = torch.tensor([ok], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if t.item() < 1 and dp.mode == P2P:
            dp.set_mode(NCCL)
            for i in range(args.warmup):
                load(i)
                step()
            barrier()
        exchange = "p2p (one fused NVLink peer-reduce + SGD kernel)" if dp.mode == P2P \
            else "nccl all-reduce + sgd"

    # ---- timed region: one event pair around the K steps (device time), a
    # fresh batch from HBM each step.  One GPU: vcnn_net_train_steps -- up to
    # 8 steps per graph launch, each staging its ring batch (the K-step chunk
    # graphs are captured in an untimed pass first)
    multi = world == 1 and not args.no_graph
    if multi:
        net.train_steps(args.steps, B, lr, mom)
        barrier()
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    launches0 = _lib.lib().vcnn_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        ev[0].record(stream)
        if multi:
            net.train_steps(args.steps, B, lr, mom)
        else:
            for i in range(args.steps):
                load(args.warmup + i)
                step()
        ev[1].record(stream)
        barrier()
    launches = _lib.lib().vcnn_launch_count() - launches0
    kps = net.kernels_per_step()
    total_s = max_over_ranks(ev[0].elapsed_time(ev[1]) / 1e3)
    value = world * B * args.steps / total_s

    # ---- e2e: host batch through the C-ABI every step ----
    e2e = None
    if not args.no_e2e:
        xin, cin, vin = net.input_tensors()
        e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
        tk = dict(cls=t_host if is_ce else None, values=None if is_ce else t_host, lr=lr,
                  momentum=mom)
        if world == 1:
            # vcnn_net_train_host_stream: every step copies its pinned host
            # batch H2D (on a copy stream, overlapping the previous step) and
            # reads its loss back D2H; events bracket the whole call
            net.train_host_stream(x_host, steps=args.warmup, **tk)
            barrier()
            e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))]
            e2e_ev[0][0].record(stream)
            net.train_host_stream(x_host, steps=args.steps, **tk)
            e2e_ev[0][1].record(stream)
        for i in range(args.steps + args.warmup if world > 1 else 0):
            if i >= args.warmup:
                e2e_ev[i - args.warmup][0].record(stream)
            if world == 1:
                net.train_step_host(x_host, cls=t_host if is_ce else None,
                                    values=None if is_ce else t_host, lr=lr, momentum=mom)
            else:
                xin[:B].copy_(x_host, non_blocking=True)
                if is_ce:
                    cin[:B].copy_(t_host, non_blocking=True)
                else:
                    vin[:B].copy_(t_host.view(B, -1), non_blocking=True)
                step()
                net.loss()  # D2H of the step's loss
            if i >= args.warmup:
                e2e_ev[i - args.warmup][1].record(stream)
        barrier()
        e2e_s = max_over_ranks(sum(a.elapsed_time(b) for a, b in e2e_ev) / 1e3)
        e2e = {"value": world * B * args.steps / e2e_s, "unit": "img/s",
               "h2d_bytes_per_step": int(x_host.numel() * 4 + t_host.numel() * 4),
               "d2h_bytes_per_step": 4, "ms_per_step": 1e3 * e2e_s / args.steps,
               "api": "vcnn_net_train_host_stream (H2D of step i+1 overlaps step i)"
               if world == 1 else "H2D + graph step + D2H loss per step"}

    if world > 1:  # the single-replica passes below must not wait on peers
        barrier()
        dp.close()
        barrier()

    # ---- per-op timing pass (eager, CUDA events around every op) ----
    pk = peaks()
    roof = None
    details = {}
    conv_gemm = None
    if rank == 0:
        rows, bd, tail_name, tot = op_timing(net, spec, B, args.steps, load, lr, mom, pk)
        top = rows[0]
        if top["bound"] == "tensor":
            roof = {"bound": "tensor", "achieved": top["tflops"], "peak": pk["tf32_tflops"],
                    "unit": "TFLOP/s", "frac": top["tflops"] / pk["tf32_tflops"]}
        else:
            roof = {"bound": "hbm", "achieved": top["gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": top["gbs"] / pk["hbm_gbs"]}
        # DRAM traffic per launch of that kernel from the committed ncu --set
        # full capture (profiles/ncu_traffic.json), when there is one
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                t = json.load(f).get(f"layer{top['layer']}.{top['op']}")
            if t and args.config == "cifar3" and B == 128:
                traffic = t["dram_bytes"]
        except (OSError, ValueError):
            pass
        kname = f"layer{top['layer']}.{top['op']}"
        if top["op"] == "loss" and tail_name:
            kname = tail_name
        roof.update({"traffic": traffic, "kernel": kname,
                     "share_of_step": top["share"], "us_per_launch": top["us"],
                     "peak_src": pk["tf32_src"] if top["bound"] == "tensor" else pk["src"]})
        step_roof_us = sum(r["roof_us"] for r in rows)
        conv_gemm = conv_gemm_rows(rows, spec, pk)
        # the same step unfused (trace kept: every conv / pool / full layer its
        # own kernels) for the reference's BreakdownTimer components (Fig. 6)
        net.set_trace(True)
        _, bd_unfused, _, _ = op_timing(net, spec, B, args.steps, load, lr, mom, pk)
        net.set_trace(False)
        details = {"ops": rows, "breakdown_s": bd, "breakdown_unfused_s": bd_unfused,
                   "step_roofline_us": step_roof_us, "eager_step_us": tot / args.steps * 1e6,
                   "peaks": pk, "conv_gemm_roofline": conv_gemm}
        # the conv GEMMs at the roofline batch (CIFAR-3 b=1024)
        if args.config == "cifar3" and not args.no_roofline_run and world == 1:
            RB = 1024
            rnet = Network(spec, RB, prec, stream=stream)
            rx, rc, rv = S.synth_bench_data(spec, RB, 11)
            rxt = torch.from_numpy(rx.reshape(RB, -1)).to(dev)
            rtt = torch.from_numpy(rc if is_ce else rv).to(dev)

            def rload(i):
                rnet.load_batch(rxt, cls=rtt if is_ce else None, values=None if is_ce else rtt)
            for i in range(3):
                rload(i)
                rnet.train_step(RB, lr, mom)
            rrows, _, _, _ = op_timing(rnet, spec, RB, 5, rload, lr, mom, pk)
            details["conv_gemm_roofline_b1024"] = conv_gemm_rows(rrows, spec, pk)
            rnet.close()
        if args.details:
            with open(args.details, "w") as f:
                json.dump(details, f, indent=1)

    # ---- the fp32-faithful mode (3xTF32) on the same workload ----
    faithful = None
    if rank == 0 and world == 1 and args.precision == "tf32" and not args.no_faithful:
        net.set_precision(S.Precision.tf32x3)
        net.enable_graph(not args.no_graph)
        for i in range(args.warmup):
            load(i)
            step()
        torch.cuda.synchronize()
        fev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        fev[0].record(stream)
        for i in range(args.steps):
            load(args.warmup + i)
            step()
        fev[1].record(stream)
        torch.cuda.synchronize()
        fsec = fev[0].elapsed_time(fev[1]) / 1e3
        faithful = {"precision": "tf32x3", "value": B * args.steps / fsec, "unit": "img/s",
                    "ms_per_step": 1e3 * fsec / args.steps,
                    "note": "fp32-faithful split-TF32 GEMMs (parity gated at 1e-5)"}
        net.set_precision(prec)

    # ---- test mode (paper Table 4): forward-only img/s, graph-replayed ----
    infer = None
    if rank == 0 and not args.no_infer:
        fs = torch.cuda.Stream()
        fs.wait_stream(stream)
        with torch.cuda.stream(fs):
            net.set_stream(fs)
            for _ in range(3):
                net.forward(B)
            fg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(fg, stream=fs):
                net.forward(B)
        net.set_stream(stream)
        stream.wait_stream(fs)
        fev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for i in range(args.warmup):
            load_copy(i)
            fg.replay()
        torch.cuda.synchronize()
        fev[0].record(stream)
        for i in range(args.steps):
            load_copy(args.warmup + i)
            fg.replay()
        fev[1].record(stream)
        torch.cuda.synchronize()
        fsec = fev[0].elapsed_time(fev[1]) / 1e3
        infer = {"metric": "test images/sec (forward only)", "value": B * args.steps / fsec,
                 "unit": "img/s", "ms_per_batch": 1e3 * fsec / args.steps, "batch": B}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(spec, B, 3, 1, seconds=args.cpu_seconds)
        if cpu:
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "img/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (Rng(8) stream, bench.cpp:29-45); random-init Glorot weights",
            "config": bench_config(args, world),
            "precision": args.precision, "graph": not args.no_graph,
            "input_pool": f"{nbatch} batches, {nbatch * x_host.numel() * 4 >> 20} MiB",
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches), "kernels_per_step": kps,
            "clocks": clk.result(),
            "step_roofline_us": details.get("step_roofline_us"),
            "conv_gemm_roofline": conv_gemm,
            "conv_gemm_roofline_b1024": details.get("conv_gemm_roofline_b1024"),
            "fp32_faithful": faithful,
            "dp_exchange": exchange,
            # BreakdownTimer components (variants.hpp:249-274, paper Fig. 6):
            # seconds per step from the event-timed eager pass
            "breakdown_ms_per_step": (
                {k: 1e3 * v / args.steps for k, v in details["breakdown_s"].items()}
                if details.get("breakdown_s") else None),
            # the same components with every layer in its own kernels (the
            # production step fuses pool into conv and the tail into one kernel)
            "breakdown_unfused_ms_per_step": (
                {k: 1e3 * v / args.steps for k, v in details["breakdown_unfused_s"].items()}
                if details.get("breakdown_unfused_s") else None),
            "infer": infer,
        }
        print(json.dumps(line))
    net.close()
    if world > 1:
        barrier()  # rank 0's single-replica passes are done on every rank's clock
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
