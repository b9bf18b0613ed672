"""CPU oracle for the continuous-sampling decode step of Infinite Sampling.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product path (`paper_2506_22950_b200/`) never imports it and the
oracle never imports the product path; they share no code.  The only shared
module is `synth/` (seeded input generators, no arithmetic of the method).

Everything here is a plain, slow, obviously-correct restatement of PAPER.md
(arXiv 2506.22950) or of a DESIGN.md reading where the paper is silent:

  sampler.py    Gumbel-max temperature sampler on Philox4x32-10 (reading R10/R11;
                PAPER.md l.382 "temperature 0.8")
  model.py      Qwen3-shaped decoder, full causal recompute per token, fp64
                (§2.1 l.106-112; Eq. 1 l.120-125)
  attention.py  plain softmax attention and the shared-prefix/suffix LSE split
                
  planner.py    Alg. 2 FPTAS grouping, Alg. 3 SJF refill, LPT, brute-force OPT
                
  simulator.py  discrete-step Alg. 1 loop: full / naive / fifo / infinite, with
                prefix phase and page-exact KV accounting (PAPER.md l.218-241,
                l.164-205)
  grpo.py       Eq. 2 and the mean-only advantage
  kv.py         KV bytes per token / per page

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
