"""BASELINE config 5 long-stream learning: C 16384, S 512, theta 8, k 40,
local inhibition r 80, whole 960x540 frames, a 100,000-frame learning stream on one GPU.

Spot parity as SURVEY §8(d) prescribes: frames 0-99 in full, then at every 10,000-frame
checkpoint the state is exported (sp_get_state, plus the duty cycles and radius with
--full) and the CPU oracle (oracle/, test infrastructure) resumes from it over the next 5
frames of the stream, which the GPU also learns as part of the stream; winners and final
permanences (and boosts / duties / radius with --full) must be bit-identical.  The oracle
checks run after the stream, one process per checkpoint.  Throughput = learning frames / the
device time of the learning calls (frame generation excluded).  One JSON line per checkpoint
and a summary line.

    python scripts/config5_stream.py [--frames 100000] [--full] [--chunk 2000]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

KW = dict(input_width=960, input_height=540, num_columns=16384, synapses_per_column=512, min_overlap=8,
          winners_set_size=40, inhibition_radius=80)
SEED_LEARN = 1001


def oracle_check(job):
    import oracle as O
    import sp_inputs
    pos, n, full, before, sdr, after = job
    cfg = O.OracleConfig(**KW, seed=42, full_learning=full, duty_cycle_period=1000, max_boost=2.0)
    ora = O.SpatialPoolerOracle(cfg, (before["idx"], before["perm"], before["boost"]))
    if full:
        ora.active_duty = before["adc"].copy()
        ora.overlap_duty = before["odc"].copy()
        ora.radius = int(before["radius"])
    t = time.time()
    res = ora.compute(sp_inputs.frames(SEED_LEARN, pos, n, 540, 960, rho=0.5), learning=True)
    bad = [i for i, r in enumerate(res) if not np.array_equal(sdr[i], O.sdr_words(r.active).view(np.int32))]
    ok = {"winners": not bad,
          "perm": bool(np.array_equal(ora.perm.view(np.uint32), after["perm"].view(np.uint32)))}
    if full:
        ok["boost"] = bool(np.array_equal(ora.boost.view(np.uint32), after["boost"].view(np.uint32)))
        ok["duties"] = bool(np.array_equal(ora.active_duty.view(np.uint32), after["adc"].view(np.uint32)) and
                            np.array_equal(ora.overlap_duty.view(np.uint32), after["odc"].view(np.uint32)))
        ok["radius"] = ora.radius == int(after["radius"])
    return {"checkpoint": pos, "frames": n, "ok": ok, "bad_frames": bad[:5],
            "mean_winners": float(np.mean([r.active.sum() for r in res])), "oracle_s": round(time.time() - t, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=100000)
    ap.add_argument("--chunk", type=int, default=2000)
    ap.add_argument("--every", type=int, default=10000)
    ap.add_argument("--head", type=int, default=100)
    ap.add_argument("--resume", type=int, default=5)
    ap.add_argument("--full", action="store_true", help="full learning (S:119(b-e)), radius adapted")
    args = ap.parse_args()
    import torch
    import paper_1608_01966_b200 as P

    flags = P.SP_FLAG_FULL_LEARNING if args.full else 0
    sp = P.SpatialPooler(**KW, max_inputs=args.chunk, flags=flags, duty_cycle_period=1000, max_boost=2.0)
    checks = {0: args.head}
    for p in range(args.every, args.frames, args.every):
        checks[p] = args.resume
    fb = torch.empty((args.chunk, 540, 960), dtype=torch.uint8, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def snap():
        idx, perm, boost = sp.get_state()
        d = {"idx": idx, "perm": perm, "boost": boost}
        if args.full:
            d["adc"], d["odc"], d["radius"], _ = sp.get_learning_state()
        return d

    jobs, dev_ms, pos, calls = [], 0.0, 0, 0
    launches0 = sp.kernel_launches()
    t0 = time.time()
    while pos < args.frames:
        nxt = min([c for c in checks if c > pos] + [args.frames])
        n = checks.get(pos, min(args.chunk, nxt - pos))
        P.synth_frames(fb[:n], pos, SEED_LEARN, 0.5)
        before = snap() if pos in checks else None
        a.record()
        sp.compute(fb[:n], learn=True)
        b.record()
        torch.cuda.synchronize()
        dev_ms += a.elapsed_time(b)
        calls += 1
        if before is not None:
            sdr = sp.winners()[0].cpu().numpy()[:n].copy()
            jobs.append((pos, n, args.full, before, sdr, snap()))
        pos += n
    wall = time.time() - t0
    info = sp.info()
    summary = {"config": "BASELINE config 5 learning stream" + (" (full learning)" if args.full else ""),
               "frames": args.frames, "device_ms": round(dev_ms, 1),
               "us_per_frame": round(dev_ms * 1e3 / args.frames, 2),
               "frames_per_s": round(args.frames / dev_ms * 1e3, 1), "learning_calls": calls,
               "kernel_launches": sp.kernel_launches() - launches0, "learn_path": P.learn_path_name(info),
               "wall_s_incl_generation_and_exports": round(wall, 1)}
    if args.full:
        summary["radius_after"] = sp.get_learning_state()[2]
    sp.close()
    del fb
    torch.cuda.empty_cache()
    with mp.get_context("fork").Pool(min(len(jobs), max(1, len(os.sched_getaffinity(0))))) as pool:
        results = pool.map(oracle_check, jobs, chunksize=1)
    for r in results:
        print(json.dumps(r), flush=True)
    summary["checkpoints"] = len(results)
    summary["all_bit_exact"] = all(all(r["ok"].values()) for r in results)
    print(json.dumps(summary), flush=True)
    return 0 if summary["all_bit_exact"] else 1


if __name__ == "__main__":
    sys.exit(main())
