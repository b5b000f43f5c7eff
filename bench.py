#!/usr/bin/env python
"""bench.py -- ME + consistency-check throughput on B200 (BASELINE.json "metric").

A step = one frame t of config 4 (1920x1080, dynamic quarter mask, float32 previous
reconstructions, K=8, S=24): for each reference d = 1..3 the whole hot path of
SURVEY.md §8(a) -- ME (qs_me_search) with the paper's NNC -> FRMC cascade fused into the call,
then PR (qs_project) -- through the C ABI.  value = frame pixels per second (Mpixel/s), the
whole job over all ranks.

  python bench.py [--gpus N --steps K --warmup W]            ours (CUDA path)
  python bench.py --impl reference ...                        the CPU oracle (rank 0 only)

N > 1 (torchrun, one rank per GPU): the frame is row-band sharded (rank r owns ~H/N rows,
SURVEY.md §8(e)); each step first exchanges the newest reference's halo rows with the
neighbouring ranks (NCCL P2P), then runs the path on its band.  Timed on the device with CUDA
events, max over ranks.  Inputs: 24 resident frames (> L2); consecutive steps use disjoint
frames (stride 4), so no step finds its inputs in L2 from the previous one.
--sequences (e.g. --config 5 --frames 12): rank r runs sequence r on the whole frame, no collective
in the step (SURVEY.md §8(e) mode (i)); value = all ranks' pixels / max rank time, weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ME+consistency-check Mpixel/s (1080p, 1/2/4/8 B200) and % of roofline"
SM_COUNT = 148
FP32_LANES_PER_SM = 128          # B200 SM: 4 SMSPs x 32 FP32 lanes (B200_PROFILING.md, blackwell guide)
SM_MAX_MHZ = 1965.0              # clocks.max.sm (B200_PROFILING.md)
# Algorithmic work per (pixel, candidate): SURVEY.md §8(d.3)/(d.4) F-b "Box" basis, 4 ops (the judged
# basis: roofline.frac); DESIGN.md's per-stage count of the same separable formulation, 8 ops (D 2 +
# H 2 + V 2 + argmin 2), is reported beside it as roofline.alt.
OPS_PER_UNIT = 4
OPS_PER_UNIT_DESIGN = 8
# uint8 configs ("bound by the integer ALU pipes"): the integer-ALU peak, measured
# per-SM issue rate of the ALU-pipe integer ops the K1i body uses (LOP3 / PRMT / VABSDIFF4 / VIMNMX,
# MEASURED_PEAKS_INT.json: 63.3 lanes per clock per SM) x 148 SMs x the max SM clock.
INT_ALU_LANES_PER_SM = 63.3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--check", default="nnc_frmc", choices=["nnc_frmc", "none"])
    ap.add_argument("--frames", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--variants", action="store_true", help="also time the CC variants (RME, RMC, FRMC, NNC->FRMC)")
    ap.add_argument("--sequences", action="store_true",
                    help="independent sequences: rank r runs sequence s = r of the config on the whole frame "
                         "(SURVEY.md 8(e) mode (i), config 5's batch; weak scaling, no collective in the step)")
    ap.add_argument("--pairs", default="refs", choices=["refs", "in_order", "streams"],
                    help="how a step runs its three (frame, reference) pairs: refs = one qs_me_search_refs call "
                         "(one launch per kernel for the three references; default), in_order = three "
                         "qs_me_search calls on one stream, streams = three calls on three streams")
    ap.add_argument("--fields", action="store_true",
                    help="refs mode: also write the three motion fields (default: projection-only, SURVEY.md 8(f) "
                         "NEXT-1 -- the vectors stay on chip and only sum / cnt are written)")
    ap.add_argument("--no-compare", action="store_true",
                    help="skip the extra timed loop that runs the same steps as three in-order qs_me_search calls")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# Clocks during the timed region (NVML, sampled every 20 ms)
# ---------------------------------------------------------------------------
_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self._h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            try:
                props = torch.cuda.get_device_properties(device_index)
                bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
                self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self._nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._h = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self._h is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._h is not None:
            self._t.join()

    def summary(self):
        if self._h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in _REASONS.items() if self.reasons & b and b != 0x1]}


# ---------------------------------------------------------------------------
# Inputs
# ---------------------------------------------------------------------------
def make_frames(cfg: int, n_frames: int, s: int = 0):
    import synth
    seq = synth.make_sequence(cfg, s)
    frames = []
    for t in range(n_frames):
        m = seq.mask(t)
        frames.append(dict(cur=(seq.frame(t) * m).astype(np.uint8), mask=m, ref=seq.ref(t)))
    return seq, frames


def step_order(n_frames: int, steps: int):
    """Frames t >= 3 (three references) visited with stride 4 so consecutive steps share no frame."""
    ts = list(range(3, n_frames))
    order = []
    for start in range(4):
        order += ts[start::4]
    return [order[i % len(order)] for i in range(steps)]


# ---------------------------------------------------------------------------
# Our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2203_09200_b200 as qs
    from paper_2203_09200_b200 import rowband
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # QS_BENCH_BACKEND=gloo: a functional check of the N > 1 code path (row bands, halo exchange staged
    # through host memory, max over ranks, the JSON line) when fewer GPUs than ranks exist -- ranks
    # share GPUs round-robin, so its numbers are not a scaling measurement; the driver's runs use NCCL.
    backend = os.environ.get("QS_BENCH_BACKEND", "nccl")
    if backend not in ("nccl", "gloo"):
        raise SystemExit(f"QS_BENCH_BACKEND={backend!r}: expected nccl or gloo")
    gpu = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        # NCCL's init lines (rank count, transports, NVLS) on stderr, so the rank count is checkable
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    cfg = synth.CONFIGS[args.config]
    W, H, K, S = cfg.w, cfg.h, cfg.K, cfg.S
    f32 = cfg.ref_f32
    if args.sequences:   # one whole sequence per rank
        band = rowband.band_of(0, 1, H, rowband.halo_rows(S, K))
        seq, frames = make_frames(args.config, args.frames, s=rank)
    else:
        # cost-balanced row bands (rowband.plan_bands: border tiles weigh 1.75 interior tiles, 1.46 for
        # float references)
        band = rowband.band_of(rank, world, H, rowband.halo_rows(S, K), S=S, K=K, f32=f32)
        seq, frames = make_frames(args.config, args.frames)
    banded = world > 1 and not args.sequences

    # Device-resident band buffers (row i = global row band.b0 + i).
    def dplane(a):
        return qs.to_plane(a[band.b0:band.b1], dev)

    dfr = []
    for fr in frames:
        ref = dplane(fr["ref"])
        if banded:      # the reconstruction exists only for owned rows until the halo exchange
            ref[:band.y0 - band.b0] = float("nan") if f32 else 0
            ref[band.y1 - band.b0:] = float("nan") if f32 else 0
        dfr.append(dict(cur=dplane(fr["cur"]), mask=dplane(fr["mask"]), ref=ref))
    if banded:          # each frame's reference halo, as it would have arrived when it was newest
        for d in dfr:
            rowband.exchange_halo(d["ref"], band)
    torch.cuda.synchronize()

    roi = qs.make_roi(W, H, band.y0, band.y1, band.b0, band.rows)
    prm = qs.make_params(K=K, S=S, min_support=8, ssd=cfg.ssd, ref_f32=f32)
    checks = qs.make_checks() if args.check == "nnc_frmc" else None
    fields = [qs.Field.alloc(band.rows, W, f32, dev) for _ in range(3)]
    wss = [qs.workspace(roi, prm, dev) for _ in range(3)]
    ws3 = qs.workspace(roi, prm, dev, n_refs=3)
    acc_s, acc_c = qs.alloc_acc(band.rows, W, dev)
    evals = torch.zeros(1, dtype=torch.int64, device=dev)

    main = torch.cuda.current_stream(dev)
    pair_streams = [torch.cuda.Stream(dev) for _ in range(3)]

    def step(t, mode):
        if banded:
            rowband.exchange_halo(dfr[t - 1]["ref"], band)
        acc_s.zero_()
        acc_c.zero_()
        if mode == "refs":       # ME + checks of the three pairs: one launch per kernel
            fr = dfr[t]
            past = [dfr[t - d] for d in (1, 2, 3)]
            qs.qs_me_search_refs(fr["cur"], fr["mask"], [x["ref"] for x in past], roi, prm,
                                 fields if args.fields else None, fuse=checks, eval_count=evals, ws=ws3,
                                 project=([x["cur"] for x in past], [x["mask"] for x in past], acc_s, acc_c))
            return
        if mode == "in_order":
            for d in (1, 2, 3):
                fr, past = dfr[t], dfr[t - d]
                qs.qs_me_search(fr["cur"], fr["mask"], past["ref"], roi, prm, fields[d - 1], fuse=checks,
                                eval_count=evals, ws=wss[d - 1])
                qs.qs_project(fields[d - 1], past["cur"], past["mask"], roi, acc_s, acc_c)
            return
        # The three (frame, reference) pairs are independent until PR: ME + checks of each pair on its
        # own stream (fills the tail waves of one pair with the next), PR serialised on the main stream.
        start = torch.cuda.Event()
        start.record(main)
        done = []
        for d in (1, 2, 3):
            ps = pair_streams[d - 1]
            ps.wait_event(start)
            fr, past = dfr[t], dfr[t - d]
            qs.qs_me_search(fr["cur"], fr["mask"], past["ref"], roi, prm, fields[d - 1], fuse=checks,
                            eval_count=evals, ws=wss[d - 1], stream=ps)
            ev = torch.cuda.Event()
            ev.record(ps)
            done.append(ev)
        for d in (1, 2, 3):
            main.wait_event(done[d - 1])
            qs.qs_project(fields[d - 1], dfr[t - d]["cur"], dfr[t - d]["mask"], roi, acc_s, acc_c)

    order = step_order(args.frames, args.warmup + args.steps)
    cmp_mode = None if args.no_compare else ("in_order" if args.pairs != "in_order" else "refs")
    for t in order[:args.warmup]:
        step(t, args.pairs)
        if cmp_mode:
            step(t, cmp_mode)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    qs.qs_profile_reset()
    qs.qs_certify_stats(reset=True)
    # The timed region: qs_profile's per-launch CUDA events are recorded on each launch's stream, so
    # in the refs and in_order modes (one stream) they time each kernel alone inside the timed region.
    qs.qs_profile_enable(True)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(gpu) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record()
        for t in order[args.warmup:]:
            step(t, args.pairs)
        t1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    qs.qs_profile_enable(False)
    rechecked = qs.qs_certify_stats(reset=True)
    ms = t0.elapsed_time(t1)
    prof = {k: qs.qs_profile_read(k) for k in qs.PROFILE_KERNELS}
    # kernels launched in the timed region: one per qs_profile scope, two for certify (scan + fix) and,
    # for float references, two for me_box (border and interior grids; QS_SPLIT=0 selects one kernel)
    split = f32 and K == 8 and os.environ.get("QS_SPLIT", "1") != "0"
    launches = sum(n for _, n in prof.values()) + prof["certify"][1] + (prof["me_box"][1] if split else 0)
    conc = None
    if cmp_mode:
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        c0.record()
        for t in order[args.warmup:]:
            step(t, cmp_mode)
        c1.record()
        torch.cuda.synchronize()
        cms = c0.elapsed_time(c1)
        if world > 1:
            tt = torch.tensor([cms], device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            cms = float(tt.item())
        n_seq_c = world if args.sequences else 1
        conc = {"pairs": cmp_mode, "value": round(n_seq_c * args.steps * W * H / (cms / 1e3) / 1e6, 3),
                "unit": "Mpixel/s", "ms_per_step": round(cms / args.steps, 4),
                "how": "same steps, timed the same way, with the other pair schedule"}
    if world > 1:
        tt = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    n_seq = world if args.sequences else 1
    value = n_seq * args.steps * W * H / (ms / 1e3) / 1e6

    # Roofline of the dominant kernel (me_box).
    me_ms, me_n = prof["me_box"]
    n_cand = (2 * S + 1) ** 2
    me_rows = min(H, band.y1 + 2) - max(0, band.y0 - 2)
    # (pixel, candidate) units of the timed region (3 pairs per step) per me_box launch
    units_per_launch = (args.steps * 3 * me_rows * W * n_cand) // me_n if me_n else 0
    achieved = OPS_PER_UNIT * units_per_launch / (me_ms / me_n / 1e3) / 1e12 if me_n else None
    peak = SM_COUNT * FP32_LANES_PER_SM * SM_MAX_MHZ * 1e6 / 1e12
    # DRAM traffic of one me_box launch of THIS config, from the ncu capture of the bench's own
    # steady-state loop with --cache-control none (profiles/me_box_traffic_c<cfg>.json); None if absent.
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"me_box_traffic_c{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # SURVEY.md 8(d.4)'s primary "pipe roofline": the busiest pipes' active fraction of me_box, from the
    # committed ncu --set full capture of this config (profiles/me_box_pipes_c<cfg>.json; None if absent).
    pipes = None
    ppath = os.path.join(ROOT, "profiles", f"me_box_pipes_c{args.config}.json")
    if os.path.exists(ppath):
        try:
            pipes = json.load(open(ppath))
        except Exception:
            pipes = None
    alt = OPS_PER_UNIT_DESIGN * units_per_launch / (me_ms / me_n / 1e3) / 1e12 if me_n else None
    roofline = {"bound": "alu", "kernel": "me_box", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "ops_per_unit": OPS_PER_UNIT, "ops_basis": "SURVEY.md 8(d.3) box ops per (pixel, candidate)",
                "units_per_launch": units_per_launch,
                "avg_launch_ms": me_ms / me_n if me_n else None,
                "share_of_step": me_ms / ms if ms else None,
                "alt": {"ops_per_unit": OPS_PER_UNIT_DESIGN, "achieved": alt,
                        "frac": (alt / peak) if alt else None, "basis": "DESIGN.md section 6 per-stage count"},
                "peak_basis": "148 SM x 128 FP32 lanes x 1965 MHz (guide unit counts and max clock)",
                "pipe": pipes}
    if not f32 and achieved:
        ipk = SM_COUNT * INT_ALU_LANES_PER_SM * SM_MAX_MHZ * 1e6 / 1e12
        roofline["int_alu"] = {"peak": ipk, "unit": "T int op/s", "frac": achieved / ipk,
                               "basis": "same 4 ops per (pixel, candidate) against the integer-ALU pipe peak "
                                        "(SURVEY.md 8(d.4) sanity ceiling; MEASURED_PEAKS_INT.json)"}
    # Second kernel of the step (epilogue: finalize + NNC -> FRMC + PR): bound by shared-memory wavefronts
    # (one per clock and SM); the wavefront count per launch is the committed ncu capture's
    # (profiles/epilogue_pipes_c<cfg>.json; absent -> no entry), the launch time is measured live here.
    ep_ms, ep_n = prof["epilogue"]
    epath = os.path.join(ROOT, "profiles", f"epilogue_pipes_c{args.config}.json")
    if ep_n and world == 1 and os.path.exists(epath):
        try:
            ep = json.load(open(epath))
            wpk = SM_COUNT * SM_MAX_MHZ * 1e6 / 1e9
            wav = ep["shared_wavefronts_per_launch"] / (ep_ms / ep_n / 1e3) / 1e9
            use = (ep["shared_wavefronts_per_launch"] - ep["bank_conflict_wavefronts_per_launch"]) \
                / (ep_ms / ep_n / 1e3) / 1e9
            roofline["second"] = {"kernel": "epilogue", "bound": "shared", "achieved": wav, "peak": wpk,
                                  "unit": "G wavefronts/s", "frac": wav / wpk,
                                  "frac_without_bank_conflicts": use / wpk,
                                  "avg_launch_ms": ep_ms / ep_n, "share_of_step": ep_ms / ms if ms else None,
                                  "peak_basis": "148 SM x 1 shared-memory wavefront per clock x 1965 MHz",
                                  "source": ep.get("source")}
        except Exception:
            pass
    kernel_ms = {k: round(v[0] / args.steps, 4) for k, v in prof.items()}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, qs, torch, dist, world, band, frames, roi, prm, checks, dev, W, H, order)

    out = None
    if rank == 0:
        out = {"metric": METRIC, "value": round(value, 3), "unit": "Mpixel/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
               "higher_is_better": True, "scaling": "weak" if args.sequences else "strong", "vs_baseline": None,
               "dtype": "f32" if f32 else ("u8 (int16x2 interior body, exact fp32 border tiles)"
                                            if os.environ.get("QS_U8_BODY") != "float" else "u8->f32(exact)"),
               "data": "synthetic",
               "config": {"workload": cfg.name, "frame": f"{W}x{H}", "K": K, "S": S, "refs": 3,
                          "mask": "dynamic" if cfg.dynamic else "fixed", "check": args.check,
                          "parallelism": (f"sequences{world}" if args.sequences else f"rowband{world}") if world > 1
                          else "single",
                          **({"backend": f"gloo functional check: {world} ranks on "
                                         f"{torch.cuda.device_count()} GPU(s), not a scaling number"}
                             if backend != "nccl" and world > 1 else {}),
                          "pairs": {"refs": "one qs_me_search_refs call per step (ME, checks and PR of the "
                                            "three references: one me_box, one epilogue launch (+ certify for "
                                            "float references)); " + ("fields written" if args.fields else
                                            "projection-only: only sum / cnt written (NEXT-1)"),
                                    "in_order": "three qs_me_search calls in order on one stream",
                                    "streams": "three qs_me_search calls on three streams"}[args.pairs],
                          "l2": f"{args.frames} resident frames (~{args.frames * W * H * (6 if f32 else 3) / 1e6:.0f} MB vs "
                                f"126 MB L2); consecutive steps use disjoint frames"},
               "roofline": roofline, "kernel_ms_per_step": kernel_ms, "gpu_launches": launches,
               "certify": {"rechecked_per_step": rechecked / args.steps,
                           "targets_per_step": round(3 * 0.75 * W * (band.y1 - band.y0)),
                           "what": "float outputs whose argmin was not certified and were recomputed in the "
                                   "definition's fp32 order (DESIGN.md 'Float certification')"} if f32 else None,
               "clocks": clk.summary(), "e2e": e2e, "compare": conc, "impl": "ours"}
        if args.variants:
            out["cc_variants_ms_per_frame"] = run_variants(qs, torch, dfr, roi, prm, fields, wss, W, H, K, S, f32)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(seq, frames, cfg)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_e2e(args, qs, torch, dist, world, band, frames, roi, prm, checks, dev, W, H, order):
    """Same metric through the C ABI with HOST inputs: each step copies its frames' planes (the
    current frame and its three references) from pinned host memory, runs the path, and reads the
    projection planes back.  The copies of step i+1 run on a second stream while step i computes
    (two slot sets, event-ordered), as a streaming deployment would; every copy is inside the
    timed region."""
    f32 = prm.ref_type == qs.QS_REF_F32

    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a[band.b0:band.b1])).pin_memory()
        return t

    host = [dict(cur=pinned(fr["cur"]), mask=pinned(fr["mask"]), ref=pinned(fr["ref"])) for fr in frames]

    def slot_set():
        return [dict(cur=qs.pitched(band.rows, W, torch.uint8, dev), mask=qs.pitched(band.rows, W, torch.uint8, dev),
                     ref=qs.pitched(band.rows, W, torch.float32 if f32 else torch.uint8, dev)) for _ in range(4)]

    sets = [slot_set(), slot_set()]
    fields = [qs.Field.alloc(band.rows, W, f32, dev) for _ in range(3)]
    wss = [qs.workspace(roi, prm, dev) for _ in range(3)]
    ws3 = qs.workspace(roi, prm, dev, n_refs=3)
    acc_s, acc_c = qs.alloc_acc(band.rows, W, dev)
    out_s = torch.empty((band.rows, W), dtype=torch.int32).pin_memory()
    out_c = torch.empty((band.rows, W), dtype=torch.uint8).pin_memory()
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    pair_streams = [torch.cuda.Stream(dev) for _ in range(3)]
    counts = {"h2d": 0, "d2h": 0}

    def issue_copies(i, ts, used_by):
        """H2D of step i's inputs into slot set i % 2 on the copy stream, after the step that last
        read that set (event used_by) is done."""
        slots = sets[i % 2]
        ev = torch.cuda.Event()
        with torch.cuda.stream(copy):
            if used_by is not None:
                copy.wait_event(used_by)
            t = ts[i]
            for j in range(4):      # slot j holds frame t - j
                src = host[t - j]
                for k in ("cur", "mask") + (("ref",) if j > 0 else ()):
                    slots[j][k].copy_(src[k], non_blocking=True)
                    counts["h2d"] += src[k].numel() * src[k].element_size()
            ev.record(copy)
        return ev

    def run(ts, start=None):
        done = [None, None]          # event: last compute that read slot set 0 / 1
        ready = issue_copies(0, ts, start)
        for i in range(len(ts)):
            slots = sets[i % 2]
            comp.wait_event(ready)
            if i + 1 < len(ts):
                ready_next = issue_copies(i + 1, ts, done[(i + 1) % 2])
            acc_s.zero_()
            acc_c.zero_()
            if args.pairs == "refs":
                qs.qs_me_search_refs(slots[0]["cur"], slots[0]["mask"], [slots[d]["ref"] for d in (1, 2, 3)], roi,
                                     prm, fields if args.fields else None, fuse=checks, ws=ws3,
                                     project=([slots[d]["cur"] for d in (1, 2, 3)],
                                              [slots[d]["mask"] for d in (1, 2, 3)], acc_s, acc_c))
            elif args.pairs == "streams":
                start = torch.cuda.Event()
                start.record(comp)
                pev = []
                for d in (1, 2, 3):
                    ps = pair_streams[d - 1]
                    ps.wait_event(start)
                    qs.qs_me_search(slots[0]["cur"], slots[0]["mask"], slots[d]["ref"], roi, prm, fields[d - 1],
                                    fuse=checks, ws=wss[d - 1], stream=ps)
                    e = torch.cuda.Event()
                    e.record(ps)
                    pev.append(e)
                for d in (1, 2, 3):
                    comp.wait_event(pev[d - 1])
                    qs.qs_project(fields[d - 1], slots[d]["cur"], slots[d]["mask"], roi, acc_s, acc_c)
            else:
                for d in (1, 2, 3):
                    qs.qs_me_search(slots[0]["cur"], slots[0]["mask"], slots[d]["ref"], roi, prm, fields[d - 1],
                                    fuse=checks, ws=wss[d - 1])
                    qs.qs_project(fields[d - 1], slots[d]["cur"], slots[d]["mask"], roi, acc_s, acc_c)
            out_s.copy_(acc_s, non_blocking=True)
            out_c.copy_(acc_c, non_blocking=True)
            counts["d2h"] += out_s.numel() * 4 + out_c.numel()
            ev = torch.cuda.Event()
            ev.record(comp)
            done[i % 2] = ev
            if i + 1 < len(ts):
                ready = ready_next

    run(order[:args.warmup])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    counts["h2d"] = counts["d2h"] = 0
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    run(order[args.warmup:], start=t0)   # the first copy waits for t0: every copy is inside the timed region
    t1.record(comp)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    n_seq = world if args.sequences else 1
    return {"value": round(n_seq * args.steps * W * H / (ms / 1e3) / 1e6, 3), "unit": "Mpixel/s",
            "h2d_bytes_per_step": counts["h2d"] // args.steps, "d2h_bytes_per_step": counts["d2h"] // args.steps,
            "ms_per_step": round(ms / args.steps, 4), "overlap": "H2D of step i+1 on a copy stream during step i"}


def run_variants(qs, torch, dfr, roi, prm, fields, wss, W, H, K, S, f32):
    """GPU analogue of Table 3's CC column: per-frame check time for each variant (3 references),
    after an untimed warm-up pass of the variant's kernels."""
    res = {}
    t = 7

    # SURVEY.md 8(f) NEXT-4 variants: NNC's second reading (R30) in the cascade, and FRMC with the
    # {0, +-(2^k - 1)} offsets extended by +-15 (valid for S >= 15)
    ext = (-15, -7, -3, -1, 0, 1, 3, 7, 15)

    def check(name, d, fr, past):
        f, ws = fields[d - 1], wss[d - 1]
        if name == "nnc_frmc":
            qs.qs_nnc(f, roi)
            qs.qs_frmc(fr["cur"], fr["mask"], past["ref"], roi, prm, f)
        elif name == "nnc_pairs_frmc":
            qs.qs_nnc_mode(f, roi, 1, qs.QS_NNC_PAIRS)
            qs.qs_frmc(fr["cur"], fr["mask"], past["ref"], roi, prm, f)
        elif name == "frmc":
            qs.qs_frmc(fr["cur"], fr["mask"], past["ref"], roi, prm, f)
        elif name == "frmc_ext15":
            qs.qs_frmc(fr["cur"], fr["mask"], past["ref"], roi, prm, f, offsets=ext)
        elif name == "rme":
            qs.qs_reverse_check(qs.QS_RME, fr["cur"], fr["mask"], past["ref"], roi, prm, f, ws=ws)
        else:
            qs.qs_reverse_check(qs.QS_RMC, fr["cur"], fr["mask"], past["ref"], roi, prm, f)

    rates = {}
    names = ("nnc_frmc", "nnc_pairs_frmc", "frmc") + (("frmc_ext15",) if S >= 15 else ()) + ("rme", "rmc")
    for name in names:
        tot = 0.0
        acc = cand = 0
        for rep in range(2):                 # rep 0: warm-up
            for d in (1, 2, 3):
                fr, past = dfr[t], dfr[t - d]
                qs.qs_me_search(fr["cur"], fr["mask"], past["ref"], roi, prm, fields[d - 1], ws=wss[d - 1])
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                check(name, d, fr, past)
                b.record()
                torch.cuda.synchronize()
                if rep:
                    tot += a.elapsed_time(b)
                    st = fields[d - 1].status
                    acc += int((st == qs.QS_ACCEPTED).sum().item())
                    cand += int((st >= qs.QS_CANDIDATE).sum().item())
        res[name] = round(tot, 3)
        rates[name] = round(acc / max(cand, 1), 4)
    res["accept_rate"] = rates       # ACCEPTED / (entries with a vector), 3 references
    return res


# ---------------------------------------------------------------------------
# The oracle: cpu_baseline (inside our line) and the --impl reference arm
# ---------------------------------------------------------------------------
def oracle_sample(frames, cfg, t, rows, threads=1):
    """The oracle on a bounded sample: output rows `rows` of frame t, references d = 1..3:
    ME -> NNC -> FRMC -> PR on those rows (timed).  The 2 halo rows of vectors NNC reads are
    computed untimed, as a full-frame run computes them once for the neighbouring rows.
    Returns the timed seconds."""
    import oracle
    K, S = cfg.K, cfg.S
    H = frames[t]["cur"].shape[0]
    y0, y1 = rows
    sec = 0.0
    s = c = None
    for d in (1, 2, 3):
        cur, msk, ref = frames[t]["cur"], frames[t]["mask"], frames[t - d]["ref"]
        kw = dict(K=K, S=S, min_support=8)
        t0 = time.perf_counter()
        f = oracle.me_search(cur, msk, ref, rows=(y0, y1), threads=threads, **kw)
        sec += time.perf_counter() - t0
        for hr in ((max(0, y0 - 2), y0), (y1, min(H, y1 + 2))):
            if hr[0] < hr[1]:
                h = oracle.me_search(cur, msk, ref, rows=hr, threads=threads, **kw)
                for k in f:
                    f[k][hr[0]:hr[1]] = h[k][hr[0]:hr[1]]
        t0 = time.perf_counter()
        f["status"] = oracle.nnc(f, 1, rows=(y0, y1))
        f["status"], _ = oracle.frmc(cur, msk, ref, f, rows=(y0, y1), threads=threads, **kw)
        s, c = oracle.project(f, frames[t - d]["cur"], frames[t - d]["mask"], s, c, rows=(y0, y1))
        sec += time.perf_counter() - t0
    return sec


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(seq, frames, cfg, rows=None):
    """The oracle timed on the box's host cores: mode 1, one thread (the paper's
    protocol, "restrict the executions to a single core"); mode 2, the OpenMP row driver
    on every host core (oracle/omp_driver.c: the same definitions, rows in parallel)."""
    import oracle
    oracle.build()
    H = cfg.h
    rows = rows or (H // 2, H // 2 + 6)
    sec = oracle_sample(frames, cfg, 3, rows)
    px = (rows[1] - rows[0]) * cfg.w
    ncores = oracle.threads_available()
    n_rows = min(H - 4, 6 * ncores)
    r2 = (max(2, H // 2 - n_rows // 2), max(2, H // 2 - n_rows // 2) + n_rows)
    sec2 = oracle_sample(frames, cfg, 3, r2, threads=ncores)
    px2 = (r2[1] - r2[0]) * cfg.w
    return {"value": round(px / sec / 1e6, 6), "unit": "Mpixel/s", "cores": 1, "kind": "oracle",
            "sample": f"frame t=3 of {cfg.name}, output rows {rows[0]}-{rows[1] - 1} ({rows[1] - rows[0]} of {H}), "
                      f"d=1..3, ME on rows +-2 (NNC halo) -> NNC -> FRMC -> PR; single-threaded C oracle",
            "seconds": round(sec, 3), "cpu_model": cpu_model(),
            "all_cores": {"value": round(px2 / sec2 / 1e6, 6), "unit": "Mpixel/s", "cores": ncores,
                          "sample": f"frame t=3, output rows {r2[0]}-{r2[1] - 1} ({n_rows} of {H}), d=1..3, same "
                                    f"chain through the OpenMP row driver on {ncores} threads",
                          "seconds": round(sec2, 3)}}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import synth
    cfg = synth.CONFIGS[args.config]
    seq, frames = make_frames(args.config, 8)
    import oracle
    oracle.build()
    H, W = cfg.h, cfg.w
    rng = np.random.default_rng(0)
    rows_per_step = 1
    def sample_rows():
        y = int(rng.integers(0, H - rows_per_step + 1))
        return (y, y + rows_per_step)
    for _ in range(args.warmup):
        oracle_sample(frames, cfg, 3 + rng.integers(0, 5), sample_rows())
    tot = 0.0
    for _ in range(args.steps):
        tot += oracle_sample(frames, cfg, 3 + int(rng.integers(0, 5)), sample_rows())
    value = args.steps * rows_per_step * W / tot / 1e6
    line = {"metric": METRIC, "value": round(value, 6), "unit": "Mpixel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * tot / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if cfg.ref_f32 else "u8", "data": "synthetic",
            "config": {"workload": cfg.name, "frame": f"{W}x{H}", "K": cfg.K, "S": cfg.S, "refs": 3,
                       "check": "nnc_frmc", "parallelism": "cpu-1-thread"},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 6), "unit": "Mpixel/s", "cores": 1, "kind": "oracle",
                             "sample": f"per step: {rows_per_step} random output row of a random frame t in 3..7, "
                                       f"d=1..3, ME rows +-2 -> NNC -> FRMC -> PR"},
            "e2e": {"value": round(value, 6), "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def main():
    args = parse()
    if args.impl == "reference":
        line = run_reference(args)
    else:
        line = run_ours(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
