"""CPU oracle for the Samoyeds hot path (arXiv 2503.10725) -- TEST INFRASTRUCTURE.

Plain, slow, obviously-correct NumPy code in fp64, written from PAPER.md.  It is
the reference the CUDA path is compared against, and nothing else:

  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it;
  * it imports nothing from ``paper_2503_10725_b200`` (the product) and the
    product never imports it -- the two share no code except the seeded input
    generators in ``synth/``.

Citations: ``P:<line>`` = /root/reference/PAPER.md line, ``S:<line>`` =
SPEC.md line (interfaces/test ideas only).  Readings of silent or garbled
passages are listed in DESIGN.md §Readings and referenced here as R<n>.

Modules
  bf16      bf16 <-> float helpers (bit level)
  fmt       (N,M,V)+2:4 format: prune, encode, decode, validate, canonical
            packing, paper Fig. 10 panel packing, byte sizes
  devlayout tcgen05 device images (A smem image, E TMEM image, index planes)
  ssmm      dual-side sparse SSMM reference + fused epilogues
  moe       routing, compaction, expert FFN, MoE layer, EP plan

Pinning status (DESIGN.md §Oracle pins): every function is pinned by
``tests/test_oracle_*.py`` except where its docstring says "parity unpinned".
"""
