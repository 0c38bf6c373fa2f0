"""Command-line front end on the GPU path, mirroring
the reference's tools/main.cpp (/root/reference/proj/tools/main.cpp):

  solve    --d --N [--restarts 20] [--seed 0] [--eps 1e-7] [--out record.json]
           [--cert-tol 1e-4] [--field complex|real]       cmd_solve   main.cpp:85-121
  sweep    --d --N-range a:b --out DIR [...]              cmd_sweep   main.cpp:198-267
  bounds   --d (--N | --N-range a:b) [--out CSV]          cmd_bounds  main.cpp:123-152
  certify  --in FRAME(.json|.csv) [--tol 1e-4]            cmd_certify main.cpp:161-196
  distortion --in FRAME [--samples N] [--seed S]          cmd_distortion main.cpp:269-279

Same output lines, CSV columns and JSON keys as the reference.  --threads is
accepted for compatibility (restarts run as a GPU batch).  --method altproj
runs the alternating-projection baseline on the GPU (baseline.py, csrc/altproj.cu).

  python -m paper_2207_06374_b200.cli solve --d 2 --N 4 --restarts 20 --seed 7 --out r.json
"""
import argparse
import json
import math
import os
import sys

from . import abi
from . import records as rec


def fmt9(v):
    """main.cpp:24-28."""
    return "%.9g" % v


def parse_range(text):
    """main.cpp:30-41."""
    if ":" not in text:
        raise ValueError("range must be of the form a:b")
    a, b = (int(x) for x in text.split(":", 1))
    if a < 1 or b < a:
        raise ValueError("range must satisfy 1 <= a <= b")
    return a, b


def _cfg(args, N):
    field = abi.REAL if args.field == "real" else abi.COMPLEX
    return abi.default_cfg(field, args.d, N, 200, eps_target=args.eps)


def run_method(args, N):
    """main.cpp:60-83."""
    if args.method == "altproj":
        if args.field == "real":
            raise NotImplementedError("method 'altproj' works on complex frames (the reference has no real mode)")
        from . import baseline
        cfg = baseline.AltProjConfig()
        result = baseline.solve_altproj(args.d, N, cfg, args.restarts, args.seed)
        return result, baseline.altproj_config_to_json(args.d, N, cfg, args.restarts, args.seed)
    if args.method != "trstmi":
        raise NotImplementedError("method '%s' is not part of this build (trstmi or altproj)" % args.method)
    cfg = _cfg(args, N)
    result = rec.solve(cfg, restarts=args.restarts, seed=args.seed)
    return result, rec.solver_config_to_json(cfg, args.restarts, args.seed)


def cmd_solve(args):
    if args.N < args.d:
        print("error: solve needs N >= d", file=sys.stderr)
        return 2
    started = rec.iso8601_utc_now()
    try:
        result, method_config = run_method(args, args.N)
    except NotImplementedError as e:
        print("error: %s" % e, file=sys.stderr)
        return 2
    finished = rec.iso8601_utc_now()
    record = rec.make_run_record(args.method, result, method_config, started, finished, args.cert_tol)
    if args.out:
        try:
            with open(args.out, "w") as f:
                f.write(json.dumps(record, indent=2) + "\n")
        except OSError:
            print("error: cannot write '%s'" % args.out, file=sys.stderr)
            return 2
    b = rec.bounds_report(args.d, args.N)
    print("d=%d N=%d method=%s coherence=%s bound=%s gap=%s" % (
        args.d, args.N, args.method, fmt9(result.best_coherence), fmt9(b["best_applicable"]),
        fmt9(result.best_coherence - b["best_applicable"])))
    return 0


def write_bounds_rows(out, d, lo, hi):
    """main.cpp:108-121."""
    out.write("N,welch,orthoplex,levenshtein,gerzon_max\n")
    for n in range(lo, hi + 1):
        b = rec.bounds_report(d, n)
        out.write("%d,%s,%s,%s,%d\n" % (n, fmt9(b["welch"]), fmt9(b["orthoplex"]) if b["orthoplex"] is not None else "",
                                        fmt9(b["levenshtein"]) if b["levenshtein"] is not None else "",
                                        b["gerzon_max"]))


def cmd_bounds(args):
    if args.N_range:
        lo, hi = parse_range(args.N_range)
    elif args.N:
        lo = hi = args.N
    else:
        print("error: bounds needs --N or --N-range", file=sys.stderr)
        return 2
    if lo < args.d:
        print("error: bounds needs N >= d", file=sys.stderr)
        return 2
    if args.out:
        with open(args.out, "w") as f:
            write_bounds_rows(f, args.d, lo, hi)
    else:
        write_bounds_rows(sys.stdout, args.d, lo, hi)
    return 0


def load_normalized(path):
    """main.cpp:154-159: frames straight from a solve pass through untouched."""
    f, d, N = rec.load_frame(path)
    if not rec.is_normalized(f, d, N, tol=1e-9):
        f = rec.normalize_columns(f, d, N)
    return f, d, N


def cmd_certify(args):
    f, d, N = load_normalized(args.inp)
    mags = rec.offdiagonal_magnitudes(f, d, N)
    mu = float(mags.max()) if mags.size and mags.max() > 0.0 else 0.0
    b = rec.bounds_report(d, N)
    tol = args.tol
    certs = [rec.certificate_to_json(c) for c in rec.certificates(f, d, N, abi.COMPLEX, tol)]
    tight, deviation = rec.check_tight(f, d, N, abi.COMPLEX, tol)
    one = rec.one_distance_report(f, d, N, abi.COMPLEX, tol)
    conj1, mub = rec.conjecture1_target(d, N), rec.mub_removal_target(d, N)
    gaps = {"to_best_bound": mu - b["best_applicable"]}
    if conj1 is not None:
        gaps["to_conjecture1"] = mu - conj1
    if mub is not None:
        gaps["to_mub_removal"] = mu - mub
    report = {"d": d, "N": N, "coherence": mu, "tolerance": tol, "bounds": rec.bounds_to_json(b),
              "tight": {"passes": tight, "deviation": deviation},
              "one_distance": rec.certificate_to_json(one), "certificates": certs,
              "targets": {"conjecture1": conj1, "mub_removal": mub}, "gaps": gaps}
    print(json.dumps(report, indent=2))
    return 0


def cmd_distortion(args):
    """main.cpp:269-279: Monte-Carlo quantisation distortion of a codebook (GPU)."""
    if args.samples < 1:
        print("error: --samples must be positive", file=sys.stderr)
        return 2
    f, d, N = load_normalized(args.inp)
    est = rec.distortion_mc(f, d, N, args.samples, args.seed)
    mags = rec.offdiagonal_magnitudes(f, d, N)
    mu = float(mags.max()) if mags.size and mags.max() > 0.0 else 0.0
    print(json.dumps({"estimate": est["estimate"], "std_error": est["std_error"], "samples": est["samples"],
                      "coherence_of_codebook": mu}, indent=2))
    return 0


def cmd_sweep(args):
    lo, hi = parse_range(args.N_range)
    if lo < args.d:
        print("error: sweep needs N >= d across the range", file=sys.stderr)
        return 2
    os.makedirs(args.out, exist_ok=True)
    rows, failures = [], 0
    for n in range(lo, hi + 1):
        try:
            started = rec.iso8601_utc_now()
            result, method_config = run_method(args, n)
            finished = rec.iso8601_utc_now()
            record = rec.make_run_record(args.method, result, method_config, started, finished, args.cert_tol)
            with open(os.path.join(args.out, "run_d%d_N%d.json" % (args.d, n)), "w") as f:
                f.write(json.dumps(record, indent=2) + "\n")
            rows.append((n, result.best_coherence))
            print("N=%d coherence=%s" % (n, fmt9(result.best_coherence)))
        except Exception as e:  # the reference reports and continues (main.cpp:230-233)
            failures += 1
            print("N=%d failed: %s" % (n, e), file=sys.stderr)
    if not rows:
        print("error: every N in the sweep failed", file=sys.stderr)
        return 1
    # point-removal correction (main.cpp:240-247)
    corrected, running = [0.0] * len(rows), math.inf
    for i in range(len(rows) - 1, -1, -1):
        running = min(running, rows[i][1])
        corrected[i] = running
    path = os.path.join(args.out, "sweep_d%d.csv" % args.d)
    with open(path, "w") as csv:
        csv.write("N,coherence,coherence_monotone,welch,orthoplex,levenshtein\n")
        for (n, mu), c in zip(rows, corrected):
            b = rec.bounds_report(args.d, n)
            csv.write("%d,%s,%s,%s,%s,%s\n" % (n, fmt9(mu), fmt9(c), fmt9(b["welch"]),
                                               fmt9(b["orthoplex"]) if b["orthoplex"] is not None else "",
                                               fmt9(b["levenshtein"]) if b["levenshtein"] is not None else ""))
    print("wrote %s (%d rows, %d failures)" % (path, len(rows), failures))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="trstmi-b200", description="TRST-MI on B200 (GPU path)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def solver_opts(p):
        p.add_argument("--d", type=int, required=True, help="ambient dimension")
        p.add_argument("--restarts", type=int, default=20)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--eps", type=float, default=1e-7, help="terminal accuracy")
        p.add_argument("--method", default="trstmi")
        p.add_argument("--threads", type=int, default=0, help="accepted for compatibility")
        p.add_argument("--cert-tol", type=float, default=rec.kDefaultCertificateTol)
        p.add_argument("--field", choices=("complex", "real"), default="complex")

    p = sub.add_parser("solve", help="optimize one (d, N) configuration")
    solver_opts(p)
    p.add_argument("--N", type=int, required=True)
    p.add_argument("--out", default="")
    p = sub.add_parser("sweep", help="solve a range of N, one record per N plus a CSV")
    solver_opts(p)
    p.add_argument("--N-range", dest="N_range", required=True)
    p.add_argument("--out", required=True)
    p = sub.add_parser("bounds", help="coherence lower bounds per N (CSV)")
    p.add_argument("--d", type=int, required=True)
    p.add_argument("--N", type=int, default=0)
    p.add_argument("--N-range", dest="N_range", default="")
    p.add_argument("--out", default="")
    p = sub.add_parser("distortion", help="Monte-Carlo quantization distortion of a codebook")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("--samples", type=int, default=1000000)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--sigma", type=float, default=1.0, help="noise variance (accepted, as the reference)")
    p.add_argument("--Es", type=float, default=1.0, help="mean symbol energy (accepted, as the reference)")
    p = sub.add_parser("certify", help="bounds, tightness and certificates of a frame file")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("--tol", type=float, default=rec.kDefaultCertificateTol)
    args = ap.parse_args(argv)
    try:
        return {"solve": cmd_solve, "sweep": cmd_sweep, "bounds": cmd_bounds, "certify": cmd_certify,
                "distortion": cmd_distortion}[args.cmd](args)
    except (ValueError, rec.FileFormatError) as e:  # usage / file errors exit 2 like the reference
        print("error: %s" % e, file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
