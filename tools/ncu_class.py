"""Per-launch ncu evidence for one training step of a bench config (1 GPU).

  run (under gpurun, ONE process):
    ncu --nvtx --nvtx-include "timed/" -k regex:"gemm_tc|conv_" --clock-control none --csv --log-file gpurun_out/X.csv \
        --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
dram__bytes_read.sum,dram__bytes_write.sum \
        python tools/ncu_class.py run c4 gpurun_out/X_prof.json
  summarise (here):
    python tools/ncu_class.py table c4 gpurun_out/X.csv gpurun_out/X_prof.json > profiles/..._tensor_table.md

`run` tunes and warms the step outside the NVTX range, then executes one
step inside the range "timed" with be.prof_enable on, and writes the
library's own launch records (kernel, M, N, K, algorithmic flops / bytes) in
issue order.  `table` matches the i-th tcgen05 kernel launch in the ncu list
with the i-th record (ncu serialises launches in issue order) and prints the
tensor-pipe utilisation per launch and the FLOP-weighted aggregate over the
compute-bound (AI ≥ ridge) launches — north_star's "≥ 60 % tensor-pipe
utilisation" gate (SURVEY §8(d) reading) — and writes the DRAM traffic per
launch of the GEMM/conv class (bench.py's roofline "traffic")."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TC_KERNELS = ("gemm_tc_kernel", "gemm_tc2_kernel", "conv_tc_kernel", "conv_small_c_kernel", "conv_stem_kernel",
              "conv_wgrad_patch_kernel", "conv_fwd_patch_kernel", "conv_wgrad_stem_kernel",
              "conv_wgrad_hankel_kernel", "conv_wgrad_hankel2_kernel", "conv_wgrad_gather_kernel")


def run(cfg_name, out):
    import torch
    import bench
    import paper_1912_01703_b200 as be
    cfg = bench.CONFIGS[cfg_name]
    stream = torch.cuda.Stream(priority=-1)
    be.init(0, stream.cuda_stream)
    be.set_compute_dtype(cfg["dtype"])
    model = bench.make_model(cfg, be)
    hb = bench.host_batch(cfg, 1)
    batch = [be.tensor(hb[0], dtype="bf16") if cfg["dtype"] == "bf16" and cfg["net"] != "ncf" else be.tensor(hb[0])]
    batch += [be.tensor(a) for a in hb[1:]]

    def step():
        return be.nn.train_step(model, batch, lr=0.01, momentum=0.9, weight_decay=1e-4, overlap_sgd=True,
                                sparse_embeddings=cfg.get("sparse", False))
    for _ in range(30):
        step()
    be.synchronize()
    be.prof_read()
    be.prof_enable(True)
    torch.cuda.nvtx.range_push("timed")
    step()
    torch.cuda.nvtx.range_pop()
    be.synchronize()
    be.prof_enable(False)
    recs = be.prof_read()
    json.dump(recs, open(out, "w"))


def _num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def table(cfg_name, csv_path, prof_path):
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    ridge = peaks["bf16_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, idi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = {}
    order = []
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        lid = r[idi]
        if lid not in launches:
            launches[lid] = {"name": r[ki]}
            order.append(lid)
        launches[lid][r[mi]] = _num(r[vi])
    recs = [r for r in json.load(open(prof_path)) if r["name"].startswith(("gemm_tc", "gemm_upd", "conv"))]
    tc = [launches[l] for l in order if any(k in launches[l]["name"] for k in TC_KERNELS)]
    print(f"# {cfg_name}: one training step under ncu (--clock-control none, serialised launches)\n")
    print(f"ncu launches in the step: {len(order)}; tcgen05 GEMM/conv launches: {len(tc)}; library records: {len(recs)}; "
          f"ridge {ridge:.0f} FLOP/B (MEASURED_PEAKS bf16_tflops / hbm_gbs)\n")
    n = min(len(tc), len(recs))
    if len(tc) != len(recs):
        print(f"WARNING: launch/record count mismatch ({len(tc)} vs {len(recs)}); matching the first {n}\n")
    print("| # | kernel | M×N×K | µs | tensor % | DRAM MB | AI (alg) | bound |")
    print("|---|---|---|---|---|---|---|---|")
    wsum = wt = 0.0
    wall = wtall = 0.0
    tot_dram = tot_us = 0.0
    for i in range(n):
        L, R = tc[i], recs[i]
        us = (L.get("gpu__time_duration.sum") or 0) / 1e3
        tp = L.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed") or 0.0
        dram = ((L.get("dram__bytes_read.sum") or 0) + (L.get("dram__bytes_write.sum") or 0))
        ai = R["flops"] / max(R["bytes"], 1)
        bound = "tensor" if ai >= ridge else "hbm"
        if bound == "tensor":
            wsum += tp * R["flops"]
            wt += R["flops"]
        wall += tp * R["flops"]
        wtall += R["flops"]
        tot_dram += dram
        tot_us += us
        import re
        m = re.search(r"(\w+)(?:<[^()]*>)?\(", L["name"])
        nm = m.group(1) if m else L["name"][:40]
        print(f"| {i} | {nm} | {R['m']}×{R['n']}×{R['k']} | {us:.1f} | {tp:.1f} | {dram / 1e6:.1f} | {ai:.0f} | {bound} |")
    print()
    if wt:
        print(f"FLOP-weighted tensor-pipe utilisation, compute-bound launches (AI ≥ ridge): **{wsum / wt:.1f} %** "
              f"over {wt / 1e12:.2f} TFLOP")
    if wtall:
        print(f"FLOP-weighted tensor-pipe utilisation, all GEMM/conv launches: {wall / wtall:.1f} % over "
              f"{wtall / 1e12:.2f} TFLOP")
    print(f"GEMM/conv class: {tot_us:.0f} µs serialised, {tot_dram / 1e6:.0f} MB DRAM, "
          f"{tot_dram / max(n, 1) / 1e6:.2f} MB per launch")
    json.dump({"kernel_class": "gemm_tc*,conv_tc*", "dram_bytes_per_launch": tot_dram / max(n, 1),
               "launches": n, "source": f"ncu dram__bytes_read+write over one {cfg_name} step ({os.path.basename(csv_path)})"},
              open(os.path.join(ROOT, "profiles", f"traffic_{cfg_name}.json"), "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        table(sys.argv[2], sys.argv[3], sys.argv[4])
