"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product path (paper_2602_00269_b200) never
imports it and fails loudly without its CUDA library.

Contents (each function cites the reference file:line it restates;
reference = /root/reference/pkg/src/speechserve/):
  weights.py  counter-based random-init mirror of csrc/init.cu + vox_api.cu
  sampler.py  restatement of sample()/apply_repetition_penalty()/
              _truncate_and_sample()/_RingWindow   (model_api.py:124-150, 311-381)
              -- PINNED against the reference's own sample() and the SPEC.md
              known-answer examples (tests/golden/sampling_golden.npz).
  paging.py   deterministic slot + KV page allocator (bit-exact page tables)
  llama.py    Llama-style backbone (prefill/decode, GQA, RoPE, RMSNorm, SiLU)
              -- parity UNPINNED by the reference (its LM is a hash stub,
              profiles.py:318-331); pinned by golden vectors we generate.
  snac.py     causal SNAC-24k-style decoder -- parity UNPINNED by the
              reference (its detokenizer emits no audio, profiles.py:333-356).
  workload.py synthetic prompt ids / request seeds (model_api.py:39-55)
"""
