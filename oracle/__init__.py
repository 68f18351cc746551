"""PipeSpec oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the verify hot
path computes, written from PAPER.md (arXiv 2505.01572).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import or execute anything under `oracle/`.  The product package
`paper_2505_01572_b200` never imports it and has no CPU fallback.

Modules:
  llama     fp64 numpy LLaMA forward, greedy argmax, AR decode, verify
            (Alg.1; greedy P:181)            pinned: HF LlamaForCausalLM,
                                                       brute-force, special cases
  buffer    token buffer O_i + KV length / page accounting (Alg.1)
                                                       pinned: SPEC S:69-81 examples
  analytic  Eqs. 1-6 and Theorem 1 (§3.3)   pinned: fixed point, limits,
                                                       Markov chain simulation
  synthetic counter-based generator + chained synthetic-alpha drafters
            (§3.3 P:123 alpha definition)
                                                       pinned: binomial 3-sigma
  protocol  virtual-clock DES of AR / sync (tiered) SD / async PipeSpec
            (Alg.1; §3.1)            pinned: losslessness == AR,
                                                       Eq.5 exact, Eq.1/3 rates

No function here is "parity unpinned" except the Fig.1/Fig.2 token-per-unit
numbers, which are not reproduced (readings R23).

The oracle shares no code with the CUDA path; the only common import is the
`synth` package (seeded data, no method arithmetic).
"""
