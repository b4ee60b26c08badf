"""CPU oracle for the NestPipe sharded-embedding step -- TEST INFRASTRUCTURE.

Plain, slow, obviously-correct numpy (fp64 accumulation) implementation of
what the hot path computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.  The
product path (``paper_2604_06956_b200``) never imports, calls or links this
package, and this package never imports the product.  The two share no code;
the only common dependency is ``workload`` (seeded input draws, no method
arithmetic).

Citations: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n (the reference
documents of arXiv 2604.06956), ``SURVEY §x`` = /root/repo/SURVEY.md.

Modules
  prf      -- counter-based table initialisation
  routing  -- sharding rule, dedup, owner bucketing, key All2All delivery,
              owner dedup, per-micro-batch send lists (S:164-172,
              S:232-250)
  step     -- the synchronous step of Definition 1 / Eq. 1-2:
              sum pooling, gradient by key, sparse SGD
  cluster  -- FWP sample clustering
  pipeline -- symbolic DBP + FWP execution with dual buffers (P:363-380,
              P:450-454) used to check Prop. 1, Prop. 2 and Corollary 1
              (P:501-548), and the six-stage negative control

Pinning status of each function is listed in DESIGN.md ("Oracle pins"); every
function here is pinned by at least one ``-m "not gpu"`` test in
tests/test_oracle_pins.py against worked examples, closed forms, brute force
or invariants -- none is "parity unpinned".
"""
