"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `compactcomm` from /root/reference/pkg/src (read-only, never copied),
drives its public API (compressors.encode / to_bytes, pipeline.encode_step /
decode_step / message_for) on seeded inputs, and writes:

  tests/golden/codec_cases.npz      per-codec KAT + random cases: input, body, decode
  tests/golden/traj_small.npz       full per-step bodies/base/fb for small trajectories
  tests/golden/traj_nm.npz          the same for the N:M block sparsifier
  tests/golden/manifest.json        digests for every case, incl. FLUX-width trajectories

The fixtures are the parity anchor for both the oracle (tests/test_oracle_golden.py)
and the CUDA path (tests/test_gpu_parity.py) on the GPU box, where the reference
is absent.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/
sys.path.insert(0, "/root/reference/pkg/src")

from compactcomm import compressors as cx  # noqa: E402
from compactcomm import linalg  # noqa: E402
from compactcomm import pipeline as pl  # noqa: E402

import synth  # noqa: E402

META = {cx.TAG_LOWRANK: 4, cx.TAG_LOWRANK_INT4: 4, cx.TAG_NMBLOCK: 4, cx.TAG_TOPK: 4}


def body_of(payload):
    blob = cx.to_bytes(payload)
    return blob[9 + META.get(payload.tag, 0):]


def spec_dict(spec):
    return {"kind": spec.kind.value, "rank": spec.rank, "iterations": spec.iterations,
            "int4_factors": spec.int4_factors, "n": spec.n, "m": spec.m,
            "keep_fraction": spec.keep_fraction}


S = cx.CompressorSpec
K = cx.CompressorKind
SIGN = S(K.SIGN1BIT)
Q2 = S(K.QUANT2BIT)

CODEC_SPECS = {
    "sign1bit": SIGN,
    "quant2bit": Q2,
    "topk0.3": S(K.TOPK, keep_fraction=0.3),
    "topk0.01": S(K.TOPK, keep_fraction=0.01),
    "lowrank-r3-f16": S(K.LOWRANK, rank=3, iterations=2),
    "lowrank-r3-int4": S(K.LOWRANK, rank=3, iterations=2, int4_factors=True),
    "nm2:4": S(K.NM_BLOCK, n=2, m=4),
    "nm1:4": S(K.NM_BLOCK, n=1, m=4),
    "nm1:2": S(K.NM_BLOCK, n=1, m=2),
    "nm4:8": S(K.NM_BLOCK, n=4, m=8),
    "nm8:16": S(K.NM_BLOCK, n=8, m=16),
    "nm5:32": S(K.NM_BLOCK, n=5, m=32),
    "nm3:5": S(K.NM_BLOCK, n=3, m=5),      # generic (non power-of-two) path
    "nm7:40": S(K.NM_BLOCK, n=7, m=40),    # generic (m > 32) path
    "nm4:4": S(K.NM_BLOCK, n=4, m=4),      # keep everything
}


def kat_inputs():
    """Hand-written inputs mirroring the reference's KATs (T/test_compressors.py)."""
    return {
        "kat_scale": np.array([[1, -1], [2, -2]], np.float32),          # :21-25
        "kat_zero": np.zeros((3, 4), np.float32),                       # :28-31
        "kat_const_mag": np.array([[3, -3, 3], [-3, 3, -3]], np.float32),  # :34-37
        "kat_zero_row": np.array([[0, 0], [2, 2]], np.float32),          # :40-42
        "kat_sign_zero": np.array([[0.0, 1.0], [-1.0, 0.0]], np.float32),  # :60-64
        "kat_tie": np.full((3, 3), 7.0, np.float32),                    # :76-82
        "kat_negzero": np.array([[-0.0, 0.0, -1.0, 2.0], [0.0, -0.0, 0.0, 0.0]], np.float32),
        "kat_zero_col": np.array([[0, 1, 2], [0, -3, 4], [0, 5, -6]], np.float32),
        "kat_tiny": np.array([[1e-38, -2e-39, 3e-45], [1e-40, 0.0, -1e-44]], np.float32),
        "kat_huge": np.array([[1e30, -3e29, 7e4], [-7.1e4, 6.6e4, 1.0]], np.float32),
        "kat_topk_hand": np.array([[3.0, 1.0], [-4.0, 0.0]], np.float32),  # :231-233
        "kat_ties": np.array([[1, -1, 1, -1, 2], [-2, 1, 1, -1, 1]], np.float32),
        "kat_nm_hand": np.array([[1.0, -5.0, 2.0, 0.0]], np.float32),   # :183-187
    }


def codec_cases():
    cases = {}
    for name, x in kat_inputs().items():
        cases[name] = x
    shapes = [(3, 5), (8, 8), (5, 12), (17, 40), (33, 128), (64, 384), (7, 1000), (1, 9), (9, 1)]
    for i, (r, c) in enumerate(shapes):
        cases[f"gauss_{r}x{c}"] = linalg.gaussian_matrix(linalg.make_rng(100 + i), r, c)
    cases["flux_64x384"] = synth.flux_like(64, 384, 1, seed=7)[0]
    cases["flux_40x3072"] = synth.flux_like(40, 3072, 1, seed=8)[0]
    return cases


def build_codec_fixture(out):
    arrays = {}
    meta = []
    for cname, x in codec_cases().items():
        x = linalg.as_matrix(x)
        arrays[f"x/{cname}"] = np.asarray(x)
        for sname, spec in CODEC_SPECS.items():
            rows, cols = x.shape
            if spec.kind == K.LOWRANK and spec.rank > min(rows, cols):
                continue
            p = cx.encode(x, spec, rng=linalg.make_rng(17))
            body = body_of(p)
            key = f"{cname}|{sname}"
            arrays[f"body/{key}"] = np.frombuffer(body, np.uint8).copy()
            dec = np.asarray(cx.decode(p))
            if dec.size <= 4096:
                arrays[f"dec/{key}"] = dec
            meta.append({"case": cname, "codec": sname, "spec": spec_dict(spec), "tag": p.tag,
                         "dec_sha256": synth.digest(dec), "rows": rows, "cols": cols, "bit_size": p.bit_size,
                         "nominal_bits": p.nominal_bits, "payload_only_bits": p.payload_only_bits,
                         "body_len": len(body)})
        # scale estimate KAT values
        sp = cx.scale_estimate(x)
        arrays[f"u/{cname}"] = sp.u
        arrays[f"v/{cname}"] = sp.v
    np.savez_compressed(os.path.join(HERE, "codec_cases.npz"), **arrays)
    out["codec_cases"] = meta


def run_traj(xs, spec, mode, warmup, rng_seed=None):
    n, c = xs[0].shape
    zero = linalg.freeze(np.zeros((n, c), np.float32))
    snd = pl.LayerState(pl.PipelineMode(mode), warmup, zero)
    rcv = pl.LayerState(pl.PipelineMode(mode), warmup, zero)
    steps = []
    for t, x in enumerate(xs, start=1):
        rng = linalg.spawn_rng(rng_seed, 5, t) if rng_seed is not None else None
        payload, rec = pl.encode_step(snd, linalg.as_matrix(x), spec, rng)
        recon = pl.decode_step(rcv, pl.message_for(t, warmup, payload))
        assert np.array_equal(recon, snd.base)
        steps.append({"payload": payload, "body": body_of(payload), "base": np.array(snd.base),
                      "fb": np.array(snd.feedback), "rec": rec})
    return steps


TRAJ_SMALL = [
    # (name, rows, cols, steps, seed, warmup)
    ("t48x256", 48, 256, 8, 21, 1),
    ("t37x100", 37, 100, 6, 22, 2),
]
TRAJ_CODECS = {"sign1bit": SIGN, "quant2bit": Q2}
NM_TRAJ_CODECS = {"nm2:4": S(K.NM_BLOCK, n=2, m=4), "nm3:5": S(K.NM_BLOCK, n=3, m=5),
                  "nm4:16": S(K.NM_BLOCK, n=4, m=16)}
MODES = ["naive", "residual_no_feedback", "residual_with_feedback"]


def build_traj_fixture(out):
    arrays = {}
    meta = []
    for name, r, c, steps, seed, warmup in TRAJ_SMALL:
        xs = synth.flux_like(r, c, steps, seed)
        for sname, spec in TRAJ_CODECS.items():
            for mode in MODES:
                key = f"{name}|{sname}|{mode}"
                res = run_traj(xs, spec, mode, warmup)
                recs = []
                for i, s in enumerate(res):
                    arrays[f"body/{key}/{i}"] = np.frombuffer(s["body"], np.uint8).copy()
                    recs.append({"base_sha256": synth.digest(s["base"]), "fb_sha256": synth.digest(s["fb"]),
                                 "step": s["rec"].step, "compression_error": s["rec"].compression_error,
                                 "bits": s["rec"].bits, "delta_hat": s["rec"].delta_hat, "tag": s["payload"].tag})
                arrays[f"base/{key}"] = res[-1]["base"]
                arrays[f"fb/{key}"] = res[-1]["fb"]
                meta.append({"key": key, "traj": name, "rows": r, "cols": c, "steps": steps, "seed": seed,
                             "warmup": warmup, "codec": sname, "mode": mode, "records": recs,
                             "inputs_sha256": synth.digest(np.stack(xs))})
    np.savez_compressed(os.path.join(HERE, "traj_small.npz"), **arrays)
    out["traj_small"] = meta


def build_nm_traj_fixture(out):
    """N:M sparsifier trajectories (all modes): per-step bodies, final base/fb."""
    arrays = {}
    meta = []
    for name, r, c, steps, seed, warmup in TRAJ_SMALL:
        xs = synth.flux_like(r, c, steps, seed)
        for sname, spec in NM_TRAJ_CODECS.items():
            for mode in MODES:
                key = f"{name}|{sname}|{mode}"
                res = run_traj(xs, spec, mode, warmup)
                recs = []
                for i, s in enumerate(res):
                    arrays[f"body/{key}/{i}"] = np.frombuffer(s["body"], np.uint8).copy()
                    recs.append({"base_sha256": synth.digest(s["base"]), "fb_sha256": synth.digest(s["fb"]),
                                 "step": s["rec"].step, "compression_error": s["rec"].compression_error,
                                 "bits": s["rec"].bits, "delta_hat": s["rec"].delta_hat, "tag": s["payload"].tag})
                arrays[f"base/{key}"] = res[-1]["base"]
                arrays[f"fb/{key}"] = res[-1]["fb"]
                meta.append({"key": key, "traj": name, "rows": r, "cols": c, "steps": steps, "seed": seed,
                             "warmup": warmup, "codec": sname, "spec": spec_dict(spec), "mode": mode,
                             "records": recs, "inputs_sha256": synth.digest(np.stack(xs))})
    # FLUX-width shard (P=8 height), 2:4, digests only
    xs = synth.flux_like(512, 3072, 4, 34)
    spec = S(K.NM_BLOCK, n=2, m=4)
    res = run_traj(xs, spec, "residual_with_feedback", 1)
    out["nm_digest"] = [{
        "key": "d512x3072|nm2:4", "rows": 512, "cols": 3072, "steps": 4, "seed": 34, "warmup": 1,
        "codec": "nm2:4", "spec": spec_dict(spec), "mode": "residual_with_feedback",
        "inputs_sha256": synth.digest(np.stack(xs)),
        "body_sha256": [synth.digest(s["body"]) for s in res],
        "base_sha256": [synth.digest(s["base"]) for s in res],
        "fb_sha256": [synth.digest(s["fb"]) for s in res],
        "records": [{"compression_error": s["rec"].compression_error, "delta_hat": s["rec"].delta_hat,
                     "bits": s["rec"].bits, "tag": s["payload"].tag} for s in res],
    }]
    np.savez_compressed(os.path.join(HERE, "traj_nm.npz"), **arrays)
    out["traj_nm"] = meta


TRAJ_DIGEST = [
    # FLUX-width shards: P=8 shard height, P=16 shard, Ulysses chunk width
    ("d512x3072", 512, 3072, 4, 31, 1, ["sign1bit", "quant2bit"]),
    ("d256x3072", 256, 3072, 5, 32, 1, ["quant2bit"]),
    ("d512x384", 512, 384, 5, 33, 1, ["sign1bit", "quant2bit"]),
]


def build_digest_fixture(out):
    meta = []
    for name, r, c, steps, seed, warmup, codecs in TRAJ_DIGEST:
        xs = synth.flux_like(r, c, steps, seed)
        for sname in codecs:
            spec = TRAJ_CODECS[sname]
            res = run_traj(xs, spec, "residual_with_feedback", warmup)
            meta.append({
                "key": f"{name}|{sname}", "rows": r, "cols": c, "steps": steps, "seed": seed, "warmup": warmup,
                "codec": sname, "mode": "residual_with_feedback",
                "inputs_sha256": synth.digest(np.stack(xs)),
                "body_sha256": [synth.digest(s["body"]) for s in res],
                "base_sha256": [synth.digest(s["base"]) for s in res],
                "fb_sha256": [synth.digest(s["fb"]) for s in res],
                "records": [{"compression_error": s["rec"].compression_error, "delta_hat": s["rec"].delta_hat,
                             "bits": s["rec"].bits} for s in res],
            })
    out["traj_digest"] = meta


def build_config1_digest(out):
    """BASELINE config 1 at full length: [4096, 3072], 2-bit, residual with feedback,
    28 steps (warmup 1), sender + receiver (pl:168-199) — per-step digests of the
    body, base and feedback.  Pins the benchmarked exchange path to the reference."""
    r, c, steps, seed, warmup = 4096, 3072, 28, 35, 1
    xs = synth.flux_like(r, c, steps, seed)
    res = run_traj(xs, Q2, "residual_with_feedback", warmup)
    out["config1_digest"] = [{
        "key": "c4096x3072|quant2bit|28", "rows": r, "cols": c, "steps": steps, "seed": seed, "warmup": warmup,
        "codec": "quant2bit", "mode": "residual_with_feedback",
        "inputs_sha256": synth.digest(np.stack(xs)),
        "body_sha256": [synth.digest(s["body"]) for s in res],
        "base_sha256": [synth.digest(s["base"]) for s in res],
        "fb_sha256": [synth.digest(s["fb"]) for s in res],
        "records": [{"compression_error": s["rec"].compression_error, "delta_hat": s["rec"].delta_hat,
                     "bits": s["rec"].bits} for s in res],
    }]


def build_topk_digest(out):
    """Top-k at a P=8-like shard: exact body digest (indices + f16 values)."""
    meta = []
    x = synth.flux_like(128, 3072, 1, seed=41)[0]
    for f in (0.01, 0.02, 0.05, 0.10):
        p = cx.encode_topk(linalg.as_matrix(x), f)
        meta.append({"rows": 128, "cols": 3072, "seed": 41, "keep_fraction": f, "k": p.kept,
                     "body_sha256": synth.digest(body_of(p))})
    out["topk_digest"] = meta


def build_lowrank_cases(out):
    """Low-rank: reference reconstruction error for tolerance-based parity."""
    meta = []
    for (r, c, seed) in ((64, 384, 51), (256, 3072, 52)):
        x = linalg.as_matrix(synth.flux_like(r, c, 1, seed)[0])
        for rank, iters, int4 in ((4, 2, False), (8, 2, False), (16, 2, False), (8, 1, False), (32, 2, True)):
            spec = S(K.LOWRANK, rank=rank, iterations=iters, int4_factors=int4)
            p = cx.encode_lowrank(x, spec, linalg.spawn_rng(seed, 5, 2))
            dec = cx.decode(p)
            err = float(np.sqrt(linalg.frob_norm_sq(dec.astype(np.float64) - x.astype(np.float64))
                                / linalg.frob_norm_sq(x)))
            meta.append({"rows": r, "cols": c, "seed": seed, "rank": rank, "iterations": iters, "int4": int4,
                         "rel_err": err, "bit_size": p.bit_size, "body_len": len(body_of(p))})
    out["lowrank"] = meta


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/compactcomm",
           "numpy": np.__version__}
    build_codec_fixture(out)
    build_traj_fixture(out)
    build_nm_traj_fixture(out)
    build_digest_fixture(out)
    build_topk_digest(out)
    build_lowrank_cases(out)
    build_config1_digest(out)
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
