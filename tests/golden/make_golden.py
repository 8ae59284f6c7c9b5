"""Generates the golden vectors in tests/golden/ from the UNMODIFIED reference
summation code (oracle/_ref/libvolpot_ref.so, built in place from
/root/reference/proj/src/{common,kernel,summation}.cpp by oracle/Makefile).

The reference ships no tests, fixtures or golden vectors, so
these fixtures pin our oracle and our GPU path to the reference's own outputs.
Inputs are stored alongside the outputs, so the fixtures do not depend on
numpy's RNG stream.  Run (in the build container, where /root/reference is
mounted):

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def main():
    ref = oracle.reference()
    ref.set_threads(1)  # the reference promises identical bytes for any count
    rng = np.random.default_rng(20221035)
    cases = {}

    # 1. Laplace FMM, random points, eps 1e-12 and 1e-6 (summation.cpp:224-348)
    src = rng.uniform(-1.0, 1.0, (3000, 2))
    tgt = rng.uniform(-0.8, 1.2, (2500, 2))
    q = rng.standard_normal(3000)
    for eps, tag in ((1e-12, "e12"), (1e-6, "e6")):
        p = ref.plan(0, 0.0, src, tgt, eps)
        cases[f"laplace_fmm_{tag}"] = dict(src=src, tgt=tgt, q=q, eps=eps, family=0, lam=0.0,
                                          levels=p.levels(), order=p.expansion_order(), out=p.apply(q))

    # 2. Laplace pairwise mode with coincident points skipped (summation.cpp:619-635)
    s2 = rng.uniform(0.0, 1.0, (1500, 2))
    t2 = np.concatenate([s2[:400], rng.uniform(0.0, 1.0, (600, 2))])
    q2 = rng.standard_normal(1500)
    p = ref.plan(0, 0.0, s2, t2, 1e-12)
    cases["laplace_pairwise"] = dict(src=s2, tgt=t2, q=q2, eps=1e-12, family=0, lam=0.0,
                                     levels=p.levels(), order=p.expansion_order(), out=p.apply(q2))

    # 3. modified Helmholtz treecode, lambda = 10 (summation.cpp:350-497)
    s3 = rng.uniform(-1.3, 1.3, (3000, 2))
    q3 = rng.standard_normal(3000)
    p = ref.plan(1, 10.0, s3, s3, 1e-12)
    cases["helm_treecode"] = dict(src=s3, tgt=s3, q=q3, eps=1e-12, family=1, lam=10.0,
                                  levels=p.levels(), order=p.expansion_order(), out=p.apply(q3))

    # 4. direct_sum, random 100 x 100 -- Laplace and K0
    s4 = rng.uniform(0.0, 1.0, (100, 2))
    t4 = rng.uniform(0.0, 1.0, (100, 2))
    q4 = rng.standard_normal(100)
    cases["direct_laplace"] = dict(src=s4, tgt=t4, q=q4, family=0, lam=0.0,
                                   out=ref.direct_sum(0, 0.0, s4, q4, t4))
    cases["direct_helm"] = dict(src=s4, tgt=t4, q=q4, family=1, lam=10.0,
                                out=ref.direct_sum(1, 10.0, s4, q4, t4))

    # 5. bessel_k0 (kernel.cpp:167-172) over both branches and the underflow
    x = np.concatenate([np.geomspace(1e-8, 2.0, 60), np.linspace(2.0, 60.0, 80),
                        np.geomspace(60.0, 900.0, 40), [2.0, 4.0, 8.0, 512.0, 1024.0]])
    cases["bessel_k0"] = dict(x=x, out=ref.bessel_k0(x))

    for name, d in cases.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, {k: (np.shape(v) if np.ndim(v) else v) for k, v in d.items()})


if __name__ == "__main__":
    main()
