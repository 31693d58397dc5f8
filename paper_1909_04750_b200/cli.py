"""Command-line entry point: the reference CLI's MICKEY rows served by the GPU.

    python -m paper_1909_04750_b200.cli gen --bits N [--seed HEX | --key HEX --iv HEX] [--lanes L]
                                            [--interleave lane|bit] [--format hex|raw] [--out FILE]
    python -m paper_1909_04750_b200.cli vectors [--file F]
    python -m paper_1909_04750_b200.cli bench [--mib M] [--repeats R] [--lanes-log2 K] [--json-out F]
    python -m paper_1909_04750_b200.cli streams --out DIR|FILE.npy [--seed HEX] [--streams N] [--stream-bits B]

`streams` writes exactly the streams `slicerng test` generates for its NIST suite (cli.py:212-231), so that the
reference's `slicerng test <files>` can judge GPU output.

Same arguments, output order and exit codes as `slicerng gen/vectors/bench`
for `--algo mickey` (pkg/src/slicerng/cli.py:102-152, 173-190, 296-369): lane-major
by default (all of lane 0's bytes, then lane 1's, ...), `--interleave bit` emits
one output word per clock.  For the same seed / key and lane count the bytes are
identical to the reference's `--impl sliced` and `--impl naive`; `--lanes` may
exceed the reference's 64 (then a bit-interleaved clock is ceil(lanes/64) 64-bit
words).  `--impl` accepts only `cuda`: there is no CPU engine in this package.  `--algo grain`
serves the reference's Grain v1 rows the same way.
"""
from __future__ import annotations

import argparse
import json
import logging
import os
import statistics
import sys
import time

import numpy as np

from . import hostmem, vectors
from .generator import MickeyGenerator
from .grain import GrainGenerator, GrainKeyIv
from .mickey import MickeyKeyIv

log = logging.getLogger("paper_1909_04750_b200")

EXIT_OK = 0
EXIT_VECTOR_MISMATCH = 3
IV_BUDGET_LOG2 = 40  # pkg/src/slicerng/mickey.py:33 (documented, not enforced)


def _parse_hex(text, nbytes=None, what="value"):
    text = text.strip().removeprefix("0x")
    try:
        data = bytes.fromhex(text)
    except ValueError as exc:
        raise ValueError(f"invalid hex for {what}: {text!r}") from exc
    if nbytes is not None and len(data) != nbytes:
        raise ValueError(f"{what} must be {nbytes} bytes, got {len(data)}")
    return data


def _init_grain(gen: GrainGenerator, args):
    """Grain material as cli._material_for builds it (cli.py:41-54): explicit key/IV (IV defaults to zero)
    or seed-derived with tag 2 (key = stream[0:10], iv = stream[10:18], seedgen.py:24-29)."""
    if args.key is not None:
        m = GrainKeyIv(_parse_hex(args.key, 10, "key"), _parse_hex(args.iv or "00" * 8, 8, "iv"))
        keys = np.tile(np.frombuffer(m.key, np.uint8), (args.lanes, 1))
        ivs = np.tile(np.frombuffer(m.iv, np.uint8), (args.lanes, 1))
    else:
        seed = _parse_hex(args.seed, 32, "seed")
        if seed == bytes(32):
            raise ValueError("all-zero master seed rejected")
        keys, ivs = gen.derive_material(seed, 0, args.lanes, algo_tag=2)
    gen.init_material(np.ascontiguousarray(keys), np.ascontiguousarray(ivs))


def _init_generator(gen: MickeyGenerator, args, lanes_padded: int):
    """Key/IV material as cli._material_for builds it (cli.py:41-54); padding lanes use zero material."""
    if args.key is not None:
        m = MickeyKeyIv(_parse_hex(args.key, 10, "key"), _parse_hex(args.iv or "", what="iv"))
        keys = np.zeros((lanes_padded, 10), np.uint8)
        ivs = np.zeros((lanes_padded, 10), np.uint8)
        keys[: args.lanes] = np.frombuffer(m.key, np.uint8)
        iv = bytes(m.iv)
        if iv:
            ivs[: args.lanes, : len(iv)] = np.frombuffer(iv, np.uint8)
        gen.init_material(keys, ivs, 8 * len(iv))
        return
    seed = _parse_hex(args.seed, 32, "seed")
    if seed == bytes(32):
        raise ValueError("all-zero master seed rejected")
    keys, ivs = gen.derive_material(seed, 0, args.lanes)
    if lanes_padded > args.lanes:
        keys = np.vstack([keys, np.zeros((lanes_padded - args.lanes, 10), np.uint8)])
        ivs = np.vstack([ivs, np.zeros((lanes_padded - args.lanes, 10), np.uint8)])
    gen.init_material(np.ascontiguousarray(keys), np.ascontiguousarray(ivs), 80)


def cmd_gen(args) -> int:
    if args.bits % 8:
        raise SystemExit("--bits must be a multiple of 8")
    nbytes = args.bits // 8
    if args.lanes < 1:
        raise SystemExit("--lanes must be at least 1")
    if args.bits > (1 << IV_BUDGET_LOG2):
        log.warning("request exceeds 2**%d bits for one key/IV; rotate material", IV_BUDGET_LOG2)
    lanes64 = (args.lanes + 63) // 64 * 64  # the reference engine is 64 lanes wide
    grain_algo = args.algo == "grain"
    with (GrainGenerator if grain_algo else MickeyGenerator)(args.device) as gen:
        if grain_algo:
            _init_grain(gen, args)   # unused lanes of the last group are the reference's unused lanes
        else:
            _init_generator(gen, args, lanes64)
        if args.interleave == "bit":
            word_bytes = lanes64 // 8
            nclocks = (nbytes + word_bytes - 1) // word_bytes
            words = gen.generate_colmajor(nclocks, stride_words=lanes64 // 32) if grain_algo else gen.generate_colmajor(nclocks)
            if grain_algo and gen.groups < lanes64 // 32:
                words[:, gen.groups:] = 0
            if args.lanes < lanes64:                # unused lanes read 0 (cli.py:125-126)
                mask = np.zeros(lanes64, np.uint8)
                mask[: args.lanes] = 1
                words &= np.packbits(mask, bitorder="little").view("<u4")[None, :]
            data = words.astype("<u4").tobytes()[:nbytes]
        else:
            per_lane = nbytes // args.lanes
            if per_lane * args.lanes != nbytes:
                raise SystemExit("--bits must split evenly across --lanes")
            rows = gen.generate_rowmajor(per_lane * 8) if per_lane else np.zeros((lanes64, 0), np.uint8)
            data = rows[: args.lanes].tobytes()
    _emit(data, args)
    return EXIT_OK


def _emit(data: bytes, args) -> None:
    if args.out:
        with open(args.out, "w" if args.format == "hex" else "wb") as fh:
            fh.write(data.hex() if args.format == "hex" else data)
        return
    if args.format == "raw":
        if sys.stdout.isatty() and not args.force_raw:
            raise SystemExit("refusing raw bytes on a terminal (use --format hex, --out FILE, or --force-raw)")
        sys.stdout.buffer.write(data)
    else:
        print(data.hex())


def cmd_vectors(args) -> int:
    algos = [args.algo] if args.algo else (["mickey"] if args.file else ["mickey", "grain"])
    bad = 0
    for algo in algos:
        records = None
        if args.file:
            with open(args.file) as fh:
                records = vectors.parse_vector_file(fh.read(), algo, args.bit_order)
        checked, failures = vectors.verify_vectors(algo, records, device=args.device)
        for f in failures:
            print(f"MISMATCH {f}")
        print(f"{algo}: {checked} vectors checked, {len(failures)} failures")
        bad += len(failures)
    return EXIT_VECTOR_MISMATCH if bad else EXIT_OK


def measure(nbytes: int, lanes: int, warmup: int = 1, repeats: int = 5, device: int = 0) -> dict:
    """Median-of-repeats record in the reference's results schema (bench.py:74-92,
    docs/conventions.md:78-84): correctness gate first (the eSTREAM vectors on every
    lane), then the keystream loop only is timed (CUDA events), like bench._timed_run."""
    checked, failures = vectors.verify_vectors("mickey", device=device)
    if failures:
        raise AssertionError("mickey/cuda failed the correctness gate: " + failures[0])
    import torch

    nclocks = max(1, nbytes * 8 // lanes)
    with MickeyGenerator(device) as gen:
        gen.init_counter(vectors.MICKEY_VECTORS[0].key, 0, lanes)
        out = torch.empty((nclocks, (lanes + 31) // 32), dtype=torch.int32, device=f"cuda:{device}")
        runs = []
        for i in range(warmup + repeats):
            gen.generate_colmajor(nclocks, out.data_ptr())
            if i >= warmup:
                runs.append(gen.last_kernel_ms * 1e-3)
    seconds = statistics.median(runs)
    total = nclocks * lanes // 8
    return {"algorithm": "mickey", "impl": "cuda", "width": lanes, "nbytes": total, "seconds": seconds,
            "gbit_per_s": total * 8 / seconds / 1e9, "runs": runs, "speedup_vs_naive": None}


def suite_streams(seed: bytes, nstreams: int, stream_bits: int, device: int = 0) -> np.ndarray:
    """The streams the reference's `slicerng test` feeds to its NIST suite (cli._suite_streams, cli.py:212-231):
    batches of 64 lanes, batch b keyed by the master seed with its first byte XORed with b, lane material from
    derive_lane_material, one mickey_sliced_words call per batch, every lane's bits packed MSB-first.  Here all
    streams come from ONE init + row-major generation on the GPU (the per-batch seeds are derived on the GPU too).
    Returns uint8[nstreams][ceil(stream_bits / 8)]; like np.packbits, a last partial byte is zero-padded."""
    if len(seed) != 32:
        raise ValueError("master seed must be 32 bytes")
    if nstreams < 1 or stream_bits < 1:
        raise ValueError("need at least one stream of at least one bit")
    nbatches = (nstreams + 63) // 64
    if nbatches > 256:
        raise ValueError("at most 256 batches of 64 streams: the batch index is folded into one seed byte (cli.py:222)")
    keys = np.empty((nstreams, 10), np.uint8)
    ivs = np.empty((nstreams, 10), np.uint8)
    nbytes = (stream_bits + 7) // 8
    with hostmem.borrow_context(MickeyGenerator, device) as gen:
        for b in range(nbatches):
            lanes = min(64, nstreams - 64 * b)
            batch_seed = bytes([seed[0] ^ b]) + seed[1:]
            if batch_seed == bytes(32):
                raise ValueError("all-zero master seed rejected")          # MasterSeed.__post_init__, seedgen.py:49-50
            gen.derive_material(batch_seed, 0, lanes, keys[64 * b: 64 * b + lanes], ivs[64 * b: 64 * b + lanes])
        rows, _ = gen.bulk_rowmajor(keys, ivs, 80, 8 * nbytes)
    if stream_bits % 8:
        rows[:, -1] &= np.uint8((0xFF << (8 - stream_bits % 8)) & 0xFF)      # np.packbits pads the tail with zeros
    return rows


def cmd_streams(args) -> int:
    """Write the suite streams: one .npy (uint8[streams][bytes]) or one raw file per stream, ready for
    `slicerng test <files>` (cli.py:183-198)."""
    rows = suite_streams(_parse_hex(args.seed, 32, "seed"), args.streams, args.stream_bits, args.device)
    if args.out.endswith(".npy"):
        np.save(args.out, rows)
    else:
        os.makedirs(args.out, exist_ok=True)
        for j, row in enumerate(rows):
            with open(os.path.join(args.out, f"stream_{j:05d}.bin"), "wb") as fh:
                fh.write(row.tobytes())
    print(f"{rows.shape[0]} stream(s) of {args.stream_bits} bits written to {args.out}")
    return EXIT_OK


def cmd_bench(args) -> int:
    rec = measure(args.mib << 20, 1 << args.lanes_log2, repeats=args.repeats, device=args.device)
    print(f"{rec['algorithm']:8s} {rec['impl']:6s} lanes={rec['width']:<9d} {rec['nbytes'] / 2**20:10.1f} MiB "
          f"{rec['seconds'] * 1e3:10.3f} ms {rec['gbit_per_s']:10.2f} Gbit/s")
    if args.json_out:
        with open(args.json_out, "w") as fh:
            json.dump({"results": [rec]}, fh, indent=2)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_1909_04750_b200",
                                description="bitsliced MICKEY 2.0 keystream on B200 (reference-compatible CLI)")
    p.add_argument("-v", "--verbose", action="store_true")
    p.add_argument("--device", type=int, default=0)
    sub = p.add_subparsers(dest="command", required=True)

    g = sub.add_parser("gen", help="generate keystream bytes")
    g.add_argument("--algo", choices=("mickey", "grain"), default="mickey")
    g.add_argument("--impl", choices=("cuda",), default="cuda")
    g.add_argument("--bits", type=int, required=True)
    g.add_argument("--seed", default="11" * 32, help="256-bit master seed (hex) for lane derivation")
    g.add_argument("--key", help="explicit key (hex); bypasses the seed")
    g.add_argument("--iv", help="explicit IV (hex)")
    g.add_argument("--lanes", type=int, default=1)
    g.add_argument("--format", choices=("raw", "hex"), default="hex")
    g.add_argument("--interleave", choices=("lane", "bit"), default="lane")
    g.add_argument("--force-raw", action="store_true")
    g.add_argument("--out")
    g.set_defaults(func=cmd_gen)

    v = sub.add_parser("vectors", help="verify embedded or file test vectors on the GPU")
    v.add_argument("--algo", choices=("mickey", "grain"))
    v.add_argument("--file", help="vector file: key=<hex> iv=<hex> ks=<hex>")
    v.add_argument("--bit-order", choices=("msb", "lsb"), default="msb")
    v.set_defaults(func=cmd_vectors)

    t = sub.add_parser("streams", help="generate the streams `slicerng test` would judge (same seeds, same lanes)")
    t.add_argument("--seed", default="11" * 32)
    t.add_argument("--streams", type=int, default=100)
    t.add_argument("--stream-bits", type=int, default=1_000_000)
    t.add_argument("--out", required=True, help="a .npy file, or a directory for one raw file per stream")
    t.set_defaults(func=cmd_streams)

    b = sub.add_parser("bench", help="GPU keystream throughput in the reference's results schema")
    b.add_argument("--mib", type=int, default=4096)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--lanes-log2", type=int, default=20)
    b.add_argument("--json-out")
    b.set_defaults(func=cmd_bench)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    logging.basicConfig(level=logging.DEBUG if args.verbose else logging.INFO,
                        format="%(levelname)s %(name)s: %(message)s")
    try:
        return args.func(args)
    except ValueError as exc:
        raise SystemExit(f"error: {exc}") from exc


if __name__ == "__main__":
    sys.exit(main())
