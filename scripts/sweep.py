#!/usr/bin/env python
"""BASELINE.json configs[4]: the single-conv-layer sweep --
kernels 3..11, channels 32..256, batch 1..1024, training and inference --
on the B200, with the reference CPU path beside it (bench.cpp run_sweep /
run_ladder / run_breakdown semantics, src/bench.cpp:195-227), written in the
reference's own report schema "vcnn-bench/1" (include/vcnn/bench.hpp:79,
src/bench.cpp:233-283) plus roofline columns.

    python scripts/sweep.py [--out profiles/r02_sweep] [--quick]

Per cell (input 32x32xC, ConvSpec{C, k, k, 1, relu}, MSE; S.single_conv):
  GPU  train: CUDA-graph replayed fwd+bwd+SGD, images/s (device events), the
       BreakdownTimer components from an event-timed eager pass, conv GEMM
       TF/s and fraction of the measured TF32 peak;
       test: graph-replayed forward.
  CPU  the reference (oracle/_ref, Executor<float>(imp6), all host threads)
       where a cell's estimated time fits the budget, else
       "n/a (time budget)"; the Imp-1..6 ladder at one cell.
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

SCHEMA = "vcnn-bench/1"
COMP = ("conv_f", "conv_b", "pool_f", "pool_b", "full_f", "full_b", "other_f", "other_b")


def env_info():
    import torch
    cpu = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"gpu": torch.cuda.get_device_name(0), "cpu": cpu, "cores": os.cpu_count(),
            "host": platform.node()}


def gpu_cell(spec, B, train, steps, pk):
    import torch
    from bench import conv_gemm_rows, op_timing
    from paper_1501_07338_b200 import spec as S
    from paper_1501_07338_b200.engine import Network
    x, _, v = S.synth_bench_data(spec, B, 8)
    net = Network(spec, B)
    xt = torch.from_numpy(x.reshape(B, -1)).cuda()
    vt = torch.from_numpy(v).cuda()

    def load(i):
        net.load_batch(xt, values=vt)
    load(0)
    st = torch.cuda.current_stream()
    rep = {}
    if train:
        net.enable_graph(True)
        for _ in range(3):
            net.train_step(B, 0.01, 0.9)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(steps):
            net.train_step(B, 0.01, 0.9)
        b.record(st)
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) / 1e3 / steps
        rows, bd, _, _ = op_timing(net, spec, B, 3, load, 0.01, 0.9, pk)
        rep["comp_seconds"] = {k: bd[k] / 3 for k in COMP}
        rep["conv_gemm"] = conv_gemm_rows(rows, spec, pk)
    else:
        for _ in range(3):
            net.forward(B)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        s2.wait_stream(st)
        with torch.cuda.stream(s2):
            net.set_stream(s2)
            net.forward(B)
            with torch.cuda.graph(g, stream=s2):
                net.forward(B)
        net.set_stream(st)
        st.wait_stream(s2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(steps):
            g.replay()
        b.record(st)
        torch.cuda.synchronize()
        sec = a.elapsed_time(b) / 1e3 / steps
    net.close()
    rep.update(images_per_sec=B / sec, median_rep_sec=sec, images_per_rep=B)
    return rep


def cpu_cell(spec, B, train, variant=6, budget=3.0):
    import ctypes as C

    import oracle_py as O
    R = O.ref()
    if R is None:
        return None, "oracle/_ref not built"
    h = R.ref_bench_create(C.byref(O.make_net(spec)), B, 8, 0.01, 0.9)
    R.ref_bench_set_variant(h, variant)
    t0 = time.perf_counter()
    R.ref_bench_step(h, int(train))  # warm-up (index-map caches)
    w = time.perf_counter() - t0
    times = []
    while sum(times) < budget and len(times) < 3:
        t = time.perf_counter()
        R.ref_bench_step(h, int(train))
        times.append(time.perf_counter() - t)
    R.ref_bench_destroy(h)
    times.sort()
    med = times[len(times) // 2]
    return {"images_per_sec": B / med, "median_rep_sec": med, "images_per_rep": B,
            "reps": len(times), "warmup": 1, "warmup_sec": w}, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sweep"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cpu-budget", type=float, default=120.0, help="total CPU seconds")
    args = ap.parse_args()
    from bench import peaks
    from paper_1501_07338_b200 import spec as S
    os.makedirs(args.out, exist_ok=True)
    pk = peaks()
    chans = (32, 64) if args.quick else (32, 64, 128, 256)
    ks = (3, 5) if args.quick else (3, 5, 7, 9, 11)
    batches = (1, 128) if args.quick else (1, 8, 64, 128, 256, 1024)
    envd = env_info()
    reports = []
    cpu_left = args.cpu_budget
    for c in chans:
        for k in ks:
            spec = S.single_conv(channels=c, k=k)
            flop_img = 2 * (32 - k + 1) ** 2 * c * c * k * k  # one conv GEMM per image
            for B in batches:
                for train in (True, False):
                    base = {"scale": f"single-conv-c{c}-k{k}", "variant": "b200",
                            "mode": "train" if train else "test", "batch": B,
                            "timestamp": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                            "environment": envd}
                    try:
                        r = gpu_cell(spec, B, train, args.steps, pk)
                        gem = 2 if train else 1  # fwd + wgrad (layer 0 has no dgrad)
                        tf = flop_img * gem * r["images_per_sec"] / 1e12
                        rep = dict(base, available=True, reps=args.steps, warmup=3, **r,
                                   conv_tflops=tf, conv_frac_of_peak=tf / pk["tf32_tflops"])
                        if "comp_seconds" in rep:
                            tot = sum(rep["comp_seconds"].values()) or 1.0
                            rep["seconds"] = rep.pop("comp_seconds")
                            rep["fraction"] = {k2: v / tot for k2, v in rep["seconds"].items()}
                    except Exception as e:  # noqa: BLE001
                        rep = dict(base, available=False, images_per_sec=None,
                                   na_reason=f"{type(e).__name__}: {e}")
                    reports.append(rep)
                    # the reference on the host: cells whose estimate fits the budget
                    est = flop_img * (3 if train else 1) * B / 20e9  # ~20 GF/s Imp-6
                    cb = dict(base, variant="imp6-cpu")
                    if est > 3.0 or cpu_left <= 0:
                        cb.update(available=False, images_per_sec=None,
                                  na_reason="n/a (time budget: estimated "
                                            f"{est:.0f} s per step on the host)")
                    else:
                        t0 = time.perf_counter()
                        cr, why = cpu_cell(spec, B, train)
                        cpu_left -= time.perf_counter() - t0
                        if cr is None:
                            cb.update(available=False, images_per_sec=None, na_reason=why)
                        else:
                            cb.update(available=True, **cr)
                    reports.append(cb)
                    print(json.dumps({k2: reports[-2].get(k2) for k2 in
                                      ("scale", "mode", "batch", "images_per_sec",
                                       "conv_tflops")}), flush=True)
    # the vectorization ladder (Imp-1..6) on the host at one cell
    spec = S.single_conv(channels=32, k=5)
    for v in range(1, 7):
        for train in (True, False):
            cr, why = cpu_cell(spec, 8, train, variant=v, budget=2.0)
            rep = {"scale": "single-conv-c32-k5", "variant": f"imp{v}-cpu",
                   "mode": "train" if train else "test", "batch": 8,
                   "timestamp": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                   "environment": envd}
            rep.update(available=cr is not None, **(cr or {"images_per_sec": None,
                                                          "na_reason": why}))
            reports.append(rep)
    doc = {"schema": SCHEMA, "peaks": pk, "reports": reports}
    with open(os.path.join(args.out, "sweep.json"), "w") as f:
        json.dump(doc, f, indent=1)
    # CSV in the reference's column order (+ roofline columns)
    with open(os.path.join(args.out, "sweep.csv"), "w") as f:
        f.write(f"# {SCHEMA}\n")
        f.write("scale,variant,mode,batch,images_per_sec," + ",".join(COMP) +
                ",reps,warmup,conv_tflops,conv_frac_of_peak\n")
        for r in reports:
            if r.get("available"):
                secs = r.get("seconds", {})
                cols = [f"{r['images_per_sec']:.6g}"] + [f"{secs.get(k, 0):.6g}" if secs else
                                                         "n/a" for k in COMP]
            else:
                cols = ["n/a"] * 9
            f.write(",".join([r["scale"], r["variant"], r["mode"], str(r["batch"])] + cols +
                             [str(r.get("reps", 0)), str(r.get("warmup", 0)),
                              f"{r.get('conv_tflops', 0):.4g}",
                              f"{r.get('conv_frac_of_peak', 0):.4g}"]) + "\n")
    print(f"wrote {len(reports)} reports to {args.out}")


if __name__ == "__main__":
    main()
