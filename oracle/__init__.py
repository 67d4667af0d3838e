"""Float64 CPU oracle for the LongLive-2.0 NVFP4 KV-cache hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import anything
under ``oracle/``.  The product path (``paper_2605_18739_b200``) never imports
it, and the oracle never imports the product path: the two share no code.

The oracle is the plain definition of what the path computes, written from
PAPER.md (arxiv 2605.18739) in the paper's order and notation:

* ``nvfp4``     -- E2M1 / E4M3 codecs and NVFP4 quantize / dequantize
                   (§2.2 Eq. 2; App. F;
                   PAPER.md:134-146 §3.2), readings Z1-Z8 of DESIGN.md.
* ``keyset``    -- the effective key set K_eff(t) of the multi-shot attention
                   sink (§4.2).
* ``attention`` -- chunk attention softmax(Q K^T / sqrt(d)) V over the
                   dequantized cache.
* ``cache``     -- the chunkwise cache driven step by step (append, evict,
                   resolve K_eff, attend).

Every function is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``)
against values the paper or mathematics fixes; see DESIGN.md §3.
"""
