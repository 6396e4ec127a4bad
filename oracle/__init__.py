"""CPU oracle for the Evoformer hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline.  The product path (``paper_2203_00854_b200``) never imports
it and fails loudly when its CUDA library is missing.

* ``evoformer_np``    - float64 numpy restatement of
                        /root/reference/pkg/src/evoplan/evoformer.py and engine.py
                        (forward oracle, every function cites file:line).
* ``evoformer_torch`` - the same algorithm in torch float64 on CPU; its autograd
                        is the gradient oracle (the reference has no backward,
                        SPEC.md:224).

The DAP schedule (dap_block.py + sharding.py) has no separate restatement: the
sharded GPU block is checked against the single-device oracle above, and its
byte ledger against the reference-generated golden ledger.

Parity is pinned: tests/test_oracle_golden.py checks these against golden
vectors produced by importing the reference itself (tests/golden/make_golden.py).
"""
