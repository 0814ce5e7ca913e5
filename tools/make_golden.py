"""Generate tests/golden/ from the reference itself (run in the dev container,
where /root/reference exists; the outputs are committed and travel to the
GPU box, which has no reference).

Inputs copied verbatim (data fixtures, not code):
  three_layer.json, greedy_counterexample.json, model_1ms.json
      <- /root/reference/proj/tests/fixtures/
  cluster1_allreduce.csv, skewed_161.json <- /root/reference/proj/data/
Outputs computed by the UNMODIFIED reference headers (oracle/_ref):
  golden.json — optimal/greedy tags and iteration-time bits (float.hex) for
  seeded random traces (ties, zeros, b = 0, tiny a included) and every
  named-model trace under traces/, plus the cluster-1 fit bits.

usage: python tools/make_golden.py
"""
from __future__ import annotations

import json
import math
import os
import random
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402

REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "tests", "golden")


def random_case(rng: random.Random, kind: str):
    if kind == "wide":  # the reference oracles.hpp:162-188 distribution, larger L
        L = rng.randint(1, 120)
        params = [int(math.exp(rng.uniform(math.log(1e2), math.log(1e8))) / 4) + 1 for _ in range(L)]
        t_b = [math.exp(rng.uniform(math.log(1e-5), math.log(1e-2))) for _ in range(L)]
        t_f = math.exp(rng.uniform(math.log(1e-4), math.log(1e-1)))
        a = math.exp(rng.uniform(math.log(1e-5), math.log(1e-2)))
        b = math.exp(rng.uniform(math.log(1e-10), math.log(1e-8)))
    else:  # ties / zeros / degenerate models (test_planner.cpp:126-155 style)
        L = rng.randint(1, 40)
        params, t_b = [], []
        for _ in range(L):
            k = rng.randrange(4)
            params.append(0 if k == 0 else (rng.randint(1, 4) if k == 1 else int(math.exp(rng.uniform(math.log(25), math.log(2.5e7))))))
            t_b.append(0.0 if rng.random() < 0.5 else math.exp(rng.uniform(math.log(1e-6), math.log(1e-2))))
        if not any(params):
            params[0] = 1
        t_f = 0.0 if rng.random() < 0.5 else math.exp(rng.uniform(math.log(1e-5), math.log(1e-1)))
        a = 1e-9 if rng.randrange(5) == 0 else math.exp(rng.uniform(math.log(1e-6), math.log(1e-1)))
        b = 0.0 if rng.randrange(4) == 0 else math.exp(rng.uniform(math.log(1e-11), math.log(1e-7)))
    return params, t_b, t_f, a, b


def ref_case(name, params, t_b, t_f, bpe, a, b):
    opt = pyoracle.ref_optimal(params, t_b, t_f, bpe, a, b)
    gr = pyoracle.ref_greedy(params, t_b, t_f, bpe, a, b)
    return {
        "name": name,
        "params": params,
        "t_b": [x.hex() for x in t_b],
        "t_f": float(t_f).hex(),
        "bpe": bpe,
        "a": float(a).hex(),
        "b": float(b).hex(),
        "optimal": "".join(map(str, opt)),
        "greedy": "".join(map(str, gr)),
        "t_optimal": pyoracle.ref_iteration_time(params, t_b, t_f, bpe, a, b, opt).hex(),
        "t_greedy": pyoracle.ref_iteration_time(params, t_b, t_f, bpe, a, b, gr).hex(),
        "t_wfbp": pyoracle.ref_iteration_time(params, t_b, t_f, bpe, a, b, [0] * len(params)).hex(),
        "t_single": pyoracle.ref_iteration_time(params, t_b, t_f, bpe, a, b, [0] + [1] * (len(params) - 1)).hex(),
    }


def main() -> None:
    assert pyoracle.REF is not None, "build oracle/_ref first: make -C oracle"
    os.makedirs(OUT, exist_ok=True)
    for f in ("three_layer.json", "greedy_counterexample.json", "model_1ms.json"):
        shutil.copy(os.path.join(REF, "tests", "fixtures", f), os.path.join(OUT, f))
    for f in ("cluster1_allreduce.csv", "skewed_161.json"):
        shutil.copy(os.path.join(REF, "data", f), os.path.join(OUT, f))

    cases = []
    rng = random.Random(20261018)
    for i in range(40):
        p, tb, tf, a, b = random_case(rng, "wide")
        cases.append(ref_case(f"wide_{i}", p, tb, tf, 4, a, b))
    for i in range(60):
        p, tb, tf, a, b = random_case(rng, "ties")
        cases.append(ref_case(f"ties_{i}", p, tb, tf, 4 if i % 3 else 2, a, b))
    # the bundled trace under the cluster-1 ring model at several N
    with open(os.path.join(OUT, "skewed_161.json")) as f:
        sk = json.load(f)
    sp = [l["params"] for l in sk["layers"]]
    stb = [l["backward_time_us"] / 1e6 for l in sk["layers"]]
    alpha, beta = 9.72e-4 / 14.0, 1.97e-9 * 8.0 / 14.0
    for n in (2, 4, 8, 16, 64, 2048):
        a = 2.0 * (n - 1.0) * alpha
        b = 2.0 * (n - 1.0) / n * beta
        cases.append(ref_case(f"skewed_161_ring_N{n}", sp, stb, sk["forward_time_us"] / 1e6, 4, a, b))
    # named-model traces (shapes from torchvision/transformers; see tools/extract_traces.py)
    tdir = os.path.join(ROOT, "traces")
    for fn in sorted(os.listdir(tdir)) if os.path.isdir(tdir) else []:
        if not fn.endswith(".json") or fn == "META.json":
            continue
        with open(os.path.join(tdir, fn)) as f:
            tr = json.load(f)
        tp = [l["params"] for l in tr["layers"]]
        ttb = [l["backward_time_us"] / 1e6 for l in tr["layers"]]
        for a, b in ((8e-6, 1.0 / 600e9), (20e-6, 1.0 / 600e9), (50e-6, 1.0 / 300e9)):
            cases.append(ref_case(f"{fn[:-5]}_a{a:g}", tp, ttb, tr["forward_time_us"] / 1e6, tr.get("bytes_per_element", 4), a, b))

    import ctypes

    a_, b_ = ctypes.c_double(), ctypes.c_double()
    rc = pyoracle.REF.ref_fit_csv(os.path.join(OUT, "cluster1_allreduce.csv").encode(), ctypes.byref(a_), ctypes.byref(b_))
    assert rc == 0
    golden = {
        "generator": "tools/make_golden.py (reference headers via oracle/_ref)",
        "cases": cases,
        "cluster1_fit": {"a": a_.value.hex(), "b": b_.value.hex()},
    }
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(golden, f, indent=0)
    print(f"wrote {len(cases)} cases to {OUT}/golden.json")


if __name__ == "__main__":
    main()
