"""Generates tests/golden/digests_full.json — SHA-256 digests of the REFERENCE's
full-size outputs at every BASELINE.json config (S=20, S=22 ER, S=24, S=26).

Run HERE (the reference sources are not on the GPU box); the JSON is committed
and tests/test_gpu_parity.py::test_full_size_digests compares the device
pipeline's arrays against it bit for bit. The reference runs through
oracle/_ref/libprpipe_ref.so (compiled from /root/reference/proj/src by
oracle/build_ref.sh) via `ref_digest_pipeline` in oracle/ref_driver.cpp, which
documents each array's byte form (int64 pairs / int64 / f64, little-endian).

    python tests/golden/make_digests.py [scale ...]     # default: 20 22 24 26

S=26 needs ~35 GB of host RAM and ~15 min on 8 threads (the reference's
run_kernel3 alone is ~7 min single-threaded).
"""
import ctypes as C
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(HERE, "digests_full.json")
# BASELINE.json configs: (scale, K0 seed, initiator name); K3 seed = K0 seed
CONFIGS = {16: (1, "graph500"), 20: (1, "graph500"), 22: (2, "uniform"), 24: (1, "graph500"), 26: (1, "graph500")}
INIT = {"graph500": O.GRAPH500, "uniform": O.UNIFORM}
ARRAYS = ("k1", "d_in", "row_offsets", "cols", "values", "ranks")


def run(scale):
    seed, iname = CONFIGS[scale]
    lib = O._ref
    emit_t = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p, C.c_int64)
    hashes = {a: hashlib.sha256() for a in ARRAYS}
    sizes = {a: 0 for a in ARRAYS}

    def emit(name, ptr, nbytes):
        name = name.decode()
        if nbytes:
            hashes[name].update((C.c_char * nbytes).from_address(ptr))
        sizes[name] += nbytes

    cb = emit_t(emit)
    f = lib.ref_digest_pipeline
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_uint64, C.POINTER(C.c_double), C.c_int, C.c_uint64, C.c_int, emit_t,
                  C.POINTER(C.c_double)]
    init = (C.c_double * 4)(*INIT[iname])
    stats = (C.c_double * 4)()
    t0 = time.time()
    rc = f(scale, seed, init, os.cpu_count() or 1, seed, 20, cb, stats)
    if rc != 0:
        raise RuntimeError(lib.ref_last_error())
    return {
        "scale": scale, "seed": seed, "initiator": iname, "k3_seed": seed, "iterations": 20, "damping": 0.85,
        "nnz_raw": int(stats[0]), "nnz_f": int(stats[1]), "max_in": int(stats[2]), "norm1": repr(stats[3]),
        "bytes": sizes, "sha256": {a: h.hexdigest() for a, h in hashes.items()},
        "generated_in_s": round(time.time() - t0, 1),
    }


def main(scales):
    if not O.have_reference():
        sys.exit("reference library not built (oracle/build_ref.sh needs /root/reference)")
    db = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for s in scales:
        rec = run(s)
        db[str(s)] = rec
        json.dump(db, open(OUT, "w"), indent=1, sort_keys=True)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or sorted(CONFIGS))
