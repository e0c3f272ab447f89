"""ORACLE -- test infrastructure only.  Plain, slow, obviously-correct CPU
reference of the rollout hot path of arXiv 2501.10709 (§3.1 MDP,
§4.2 VecEnv reset/step/reward, §4.3 T x N x D samples, §5.2 ensembles, §6.1 /
Eq. 6 metrics), written from the paper in the paper's order and notation.

Rules:
* float64 everywhere (pure Python ``float`` = IEEE binary64, never contracted
  into FMA); NumPy is used only as array storage and for the float64 matmul of
  the MLP, which is cross-checked against explicit loops in the pins.
* No import of, and no shared code with, the CUDA package
  ``paper_2501_10709_b200``.  Inputs come from ``synth`` (seeded generators
  that hold none of the method's arithmetic).
* Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import this package.

Modules: ``quant`` (bf16 rounding, round-half-away), ``stock`` (stock env),
``crypto`` (crypto env), ``mlp`` (policy / Q forward), ``policy`` (action
sampling, ensemble), ``metrics`` (episode metrics), ``philox`` (counter-based
RNG for production-mode noise), ``rollout`` (drivers).
"""
