"""Seeded synthetic INPUT generators shared by the oracle and the CUDA path.

This package holds none of the method's arithmetic (no env step, no MLP, no
sampling rule, no metric).  It only produces the data both sides consume:

* ``market``  -- stock OHLCV + technical-indicator tensors (GBM close prices)
                 and the crypto limit-order-book + factor rows.
* ``policy``  -- Kaiming-uniform bf16 weights for the policy / Q networks.
* ``inputs``  -- seeded integer share actions and supplied N(0,1) noise.

Everything is NumPy with ``np.random.Generator(PCG64(seed))``; identical seeds
give identical bytes.  Stand-ins for the paper's datasets:
the DJIA-30 daily OHLCV and the BTC second-level LOB are not available, so
BASELINE.json configs[0..4] define synthetic data of the same shape.
"""
