"""bench.py -- MRFMap hot path on B200: ray-voxel message updates/s (BASELINE.json metric).

One step = the whole hot path over one batch of synthetic input:
  reset; add_frame x F (raygen + DDA count, scan, DDA fill); bp_iterate(n) (transpose build,
  then n x [K5 ray messages, K6 voxel reduction, (K7 all-reduce)]); marginals.
Units per step = E * n (message updates), E = incidences of all ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config frames30] [--impl ours|reference]

N > 1: one rank per GPU, rays sharded by pixel row (v % world == rank) with an NCCL all-reduce
of the int64 voxel sums of the touched tiles every iteration.  Launched by the driver under
torch.distributed.run; `--gpus N` without WORLD_SIZE in the environment re-launches itself
that way (N ranks on 127.0.0.1).  NCCL's INFO lines (communicator set-up, NVLS) go to
gpurun_out/nccl.<host>.<pid>.log unless NCCL_DEBUG is set.  `--dry-run` exercises the launch
and rank plumbing on CPU (gloo, no kernels).
--impl reference: the fp64 CPU oracle (oracle/) timed on the host cores on a bounded sample
of the same workload (this tier has no reference implementation to install).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ray-voxel message updates/sec"
UNIT = "updates/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- reference arm

def _oracle_sample(w, max_frames=1, messages="per-ray", threads=None, n_iter=None):
    """The oracle as it stands on a bounded sample: the first `max_frames` frames of the
    workload, graph build + n iterations, on `threads` OpenMP threads (None: all cores).
    Returns (updates, seconds, E, threads used)."""
    import oracle
    n_iter = w.n_iter if n_iter is None else n_iter
    used = _cores() if threads is None else int(threads)
    oracle.set_num_threads(used)
    try:
        p = oracle.Params.from_workload(w)
        t0 = time.perf_counter()
        g = oracle.build_graph(p, w.frames[:max_frames])
        if messages == "keyframe-avg":
            oracle.kf_bp(p, g, n_iter, F=max_frames)
        else:
            oracle.bp(p, g, n_iter)
        dt = time.perf_counter() - t0
    finally:
        oracle.set_num_threads(_cores())
    return g.E * n_iter, dt, g.E, used


def cpu_baseline(w, config, messages):
    """the fp64 oracle on the host, at all cores (first 5 frames of the workload)
    and at 1 thread (first frame), graph build + the workload's iterations, as it stands."""
    nf = min(5, len(w.frames))
    u, dt, E, used = _oracle_sample(w, nf, messages)
    u1, dt1, E1, _ = _oracle_sample(w, 1, messages, threads=1)
    v, v1 = u / dt, u1 / dt1
    return {"value": v, "unit": UNIT, "cores": used, "kind": "oracle", "cpu": _cpu_model(),
            "ns_per_incidence_iteration": 1e9 / v,
            "sample": f"subset: first {nf} of {len(w.frames)} frames of {config} (E={E}), graph build + "
                      f"{w.n_iter} BP iterations, fp64, {used} OpenMP threads",
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "ns_per_incidence_iteration": 1e9 / v1,
                              "sample": f"subset: first frame of {config} (E={E1}), graph build + "
                                        f"{w.n_iter} BP iterations, fp64, 1 thread"}}


def _workload(args):
    import synth
    w = synth.make_workload(args.config)
    if args.noise == "patch":  # the learnt per-patch sensor model (R25) over the config's frames
        H, W = w.frames[0].depth.shape
        w.patch = synth.patch_noise_model(W, H, w.seed, 20, w.sigma_c)
    return w


def run_reference(args, rank, world):
    import synth
    if rank != 0:
        return
    w = _workload(args)
    for _ in range(args.warmup):
        _oracle_sample(w, 1, args.messages)
    tot_u = tot_t = 0.0
    for _ in range(args.steps):
        u, dt, E, cores = _oracle_sample(w, 1, args.messages)
        tot_u += u
        tot_t += dt
    v = tot_u / tot_t
    sample = (f"subset: first frame of {args.config} (E={E}), graph build + {w.n_iter} BP iterations per step, "
              f"fp64, {cores} OpenMP threads ({_cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "sample": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": _cpu_model(), "ns_per_incidence_iteration": 1e9 / v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import synth
    import paper_2006_03512_b200 as pkg

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = _workload(args)
    n_iter = w.n_iter if args.iters is None else args.iters

    kw = {}
    if world > 1:
        ids = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        kw = dict(rank=rank, world=world, comm=pkg.MRF_COMM_NCCL, nccl_id=ids[0])
    stream = torch.cuda.current_stream(dev)
    # The 0.02 m configs exceed one ctx's 2^31 incidence slots on a single GPU: there the GPU
    # holds several emulated ranks (dist.EmulatedRanks) whose per-iteration int64 partials are
    # summed on the device.
    emulate = args.emulate_ranks if args.emulate_ranks is not None else (
        4 if (world == 1 and args.config in ("frames100", "sweep300") and not args.bricks) else 1)
    if args.messages == "keyframe-avg":
        assert world == 1 and emulate == 1, "keyframe averages are single-rank (one ctx, < 2^31 incidences)"
    if emulate > 1:
        assert world == 1, "--emulate-ranks is a single-GPU mode"
        from paper_2006_03512_b200.dist import EmulatedRanks
        m = EmulatedRanks(w, emulate, stream.cuda_stream)
    else:
        m = pkg.MRFMap.from_workload(w, **kw)
        m.set_stream(stream.cuda_stream)
        if args.messages == "keyframe-avg":  # NEXT #3: the paper's per-keyframe average messages
            m.set_message_mode(pkg.MRF_MSG_KEYFRAME_AVG)
    if args.bricks:  # NEXT #4: brick allocation around the depth points + empty-skip walks
        for mm in (m.maps if emulate > 1 else [m]):
            mm.set_sparse_bricks(args.bricks)
    if args.matrix_free:  # NEXT #1: keep only lambda + tile runs, re-walk per chunk of frames
        for mm in (m.maps if emulate > 1 else [m]):
            mm.set_matrix_free(args.matrix_free)

    depth_dev = [torch.from_numpy(fr.depth).to(dev) for fr in w.frames]
    depth_host = [torch.from_numpy(fr.depth).pin_memory() for fr in w.frames]
    marg_dev = torch.empty(w.n_voxels, dtype=torch.float32, device=dev)
    marg_host = torch.empty(w.n_voxels, dtype=torch.float32).pin_memory()

    def step(host_io=False):
        m.reset()
        for fr, dd, dh in zip(w.frames, depth_dev, depth_host):
            m.add_frame(dh if host_io else dd, fr.K, fr.T_wc)
        m.bp_iterate(n_iter)
        if host_io:
            m.marginals(marg_host.numpy())
        else:
            m.marginals(marg_dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up (also sizes every buffer)
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    sizes = m.graph_sizes()
    E_local = sizes["E"]
    t = torch.tensor([E_local, sizes["n_rays"]], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(t)
    E_all, R_all = int(t[0]), int(t[1])

    # ---- timed region (device-resident inputs)
    m.set_profiling(True)
    m.profile_read()
    launches0 = m.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    launches = m.launch_count() - launches0
    prof = m.profile_read()
    m.set_profiling(False)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t)
    units = E_all * n_iter * args.steps
    value = units / (ms / 1e3)

    # ---- end to end through the public API: host depth in, host marginals out
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        step(host_io=True)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms_e2e = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_e2e, op=dist.ReduceOp.MAX)
    e2e_value = E_all * n_iter * e2e_steps / (float(ms_e2e) / 1e3)
    h2d = sum(fr.depth.nbytes for fr in w.frames)
    d2h = w.n_voxels * 4

    # ---- roofline of the dominant kernel (one launch group = one BP iteration over all classes)
    # roofline.frac counts the METHOD's bytes, SURVEY §8(d)'s canonical model:
    #   K5: vid 4 + off_q 2 + lambda read 4 + lambda write 4 = 14 B per incidence, + T gather 8 per voxel
    #   K6: tr 4 + lambda 4 = 8 B per incidence, + T write 8 per voxel
    # This design's own bytes (K5 reads a 4-byte log nu instead of the 2-byte off_q; K6 reads 16 B
    # per tile run instead of tr) are reported beside them under "design_bytes".
    peak, peak_kind = _peaks()
    V = w.n_voxels
    lay = m.layout_sizes()
    n_runs = lay["n_runs"]
    n_k5, ms_k5 = prof["ray_messages"]
    n_k6, ms_k6 = prof["voxel_sum"]
    per_iter_k5 = ms_k5 / max(1, args.steps * n_iter)
    per_iter_k6 = ms_k6 / max(1, args.steps * n_iter)
    bytes_k5 = 14 * E_local + 8 * V
    bytes_k6 = 8 * E_local + 8 * V
    dbytes_k5 = 16 * E_local + 8 * V             # this design
    # K6 path: the pixel-block hash reduction (K6b, default for per-ray messages over a stored
    # graph: vid + lambda of every slot of the rows, padding included) or the tile-run K6
    k6_path = m.k6_path()
    dbytes_k6 = (8 * lay["n_slots"] + 8 * V) if k6_path == "block" else (4 * E_local + 16 * n_runs + 8 * V)
    gbs = lambda b, t: b / (t / 1e3) / 1e9 if t > 0 else 0.0
    ach_k5, ach_k6 = gbs(bytes_k5, per_iter_k5), gbs(bytes_k6, per_iter_k6)
    ach_bp = gbs(bytes_k5 + bytes_k6, per_iter_k5 + per_iter_k6)
    dach_k5, dach_k6 = gbs(dbytes_k5, per_iter_k5), gbs(dbytes_k6, per_iter_k6)
    dach_bp = gbs(dbytes_k5 + dbytes_k6, per_iter_k5 + per_iter_k6)
    dominant = "ray_messages" if ms_k5 >= ms_k6 else "voxel_sum"
    ach = ach_k5 if dominant == "ray_messages" else ach_k6
    # ncu DRAM bytes per launch (one --set full capture of this workload, profiles/ncu_summary.json)
    # over the live kernel times: SURVEY §8(d)'s reporting rule 1 (achieved DRAM GB/s / peak)
    traffic_of = {}
    prof_json = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_json):
        try:
            d = json.load(open(prof_json))
            for name, k in d.get("kernels", {}).items():
                if (k.get("config") == args.config and k.get("E") == E_local and args.messages == "per-ray"
                        and args.noise == "lut"):
                    traffic_of[name] = k.get("dram_bytes_per_launch")
        except Exception:
            pass
    traffic = traffic_of.get(dominant)
    dram = {}
    if "ray_messages" in traffic_of and "voxel_sum" in traffic_of:
        t5, t6 = traffic_of["ray_messages"], traffic_of["voxel_sum"]
        dram = {"k5_dram_frac": gbs(t5, per_iter_k5) / peak, "k6_dram_frac": gbs(t6, per_iter_k6) / peak,
                "bp_iteration_dram_frac": gbs(t5 + t6, per_iter_k5 + per_iter_k6) / peak}

    if rank == 0:
        kernel_ms = {k: round(v[1] / max(1, args.steps), 4) for k, v in prof.items() if v[0]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": args.config, "frames": len(w.frames), "bp_iterations": n_iter,
                       "messages": args.messages, "bricks": args.bricks, "matrix_free": args.matrix_free,
                       "noise": args.noise,
                       "incidences": E_all, "rays": R_all, "voxels": V, "grid": list(w.dims), "res_m": w.res,
                       "parallelism": (f"rays sharded by pixel row over {world} GPU(s)" if world > 1 else
                                       f"1 GPU, {emulate} emulated ranks (device-side int64 reduce)" if emulate > 1
                                       else "1 GPU"),
                       "l2": f"inputs larger than L2: messages {4 * E_all / 1e9:.2f} GB, graph {10 * E_all / 1e9:.2f} GB"},
            "ms_per_bp_iteration": (ms_k5 + ms_k6 + prof["allreduce"][1]) / max(1, args.steps * n_iter),
            "kernel_ms_per_step": kernel_ms,
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_model": "SURVEY §8(d): K5 14 B/incidence + 8 B/voxel, K6 8 B/incidence + 8 B/voxel",
                         "algorithmic_bytes_per_launch": bytes_k5 if dominant == "ray_messages" else bytes_k6,
                         "k5_frac": ach_k5 / peak, "k6_frac": ach_k6 / peak,
                         "bp_iteration_frac": ach_bp / peak,
                         "k6_path": k6_path,
                         "design_bytes": {"model": "K5 16 B/incidence (log nu stored) + 8 B/voxel; " +
                                                   ("K6b 8 B/slot (vid + lambda, padding included) + 8 B/voxel"
                                                    if k6_path == "block" else
                                                    "K6 4 B/incidence + 16 B/tile run + 8 B/voxel"),
                                          "k5_frac": dach_k5 / peak, "k6_frac": dach_k6 / peak,
                                          "bp_iteration_frac": dach_bp / peak},
                         "ms_k5": per_iter_k5, "ms_k6": per_iter_k6, "tile_runs": n_runs, **dram},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, args.config, args.messages)
        print(json.dumps(line), flush=True)
    m.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="frames30")
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--matrix-free", type=int, default=0,
                    help="frames per re-walked chunk (NEXT #1: only messages + tile runs stored; 0 = stored graph)")
    ap.add_argument("--bricks", type=int, default=0,
                    help="sparse-brick map with B^3 bricks (P:203-205; 0 = dense, the north_star graph)")
    ap.add_argument("--messages", default="per-ray", choices=["per-ray", "keyframe-avg"],
                    help="message model: exact per-ray messages (north_star) or per-keyframe averages (P:200)")
    ap.add_argument("--noise", default="lut", choices=["lut", "patch"],
                    help="sensor model: the global table (north_star) or learnt per-patch polynomials (P:207-230)")
    ap.add_argument("--emulate-ranks", type=int, default=None,
                    help="ranks emulated on the one GPU (default: 4 for the 0.02 m configs, else 1)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / rank plumbing only (gloo on CPU, no kernels): one JSON line from rank 0")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} ranks", file=sys.stderr)
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        _nccl_log_env()
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _self_launch(n):
    """`--gpus N` outside torch.distributed.run: re-launch this script as N ranks (one per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def _nccl_log_env():
    """Keep NCCL's INFO lines (communicator set-up: rings, NVLS, P2P/NVLink transports) in a file
    per rank, out of stdout (rank 0's stdout carries the one JSON line)."""
    if "NCCL_DEBUG" in os.environ:
        return None
    d = os.path.join(ROOT, "gpurun_out")
    os.makedirs(d, exist_ok=True)
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    os.environ["NCCL_DEBUG_FILE"] = os.path.join(d, "nccl.%h.%p.log")
    return os.environ["NCCL_DEBUG_FILE"]


def run_dry(args, rank, world):
    """The N-rank plumbing without a GPU: gloo process group, the row sharding of the workload's
    frames (v % world == rank), the max-over-ranks timing reduction; rank 0 prints one line."""
    import torch
    import torch.distributed as dist

    import synth
    from paper_2006_03512_b200.dist import owned_rows

    if world > 1:
        dist.init_process_group("gloo")
    w = synth.make_workload(args.config)
    t0 = time.perf_counter()
    pix = sum(len(owned_rows(fr.height, rank, world)) * fr.width for fr in w.frames)
    t = torch.tensor([1, pix, rank], dtype=torch.int64)
    ms = torch.tensor([1e3 * (time.perf_counter() - t0)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks": int(t[0]), "rank_sum": int(t[2]),
                          "pixels": int(t[1]), "pixels_expected": sum(fr.height * fr.width for fr in w.frames),
                          "ms_max_over_ranks": float(ms), "config": {"workload": args.config}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
