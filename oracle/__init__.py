"""CPU oracle for the RLHFSpec verification hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference implementations written from the paper
(/root/reference/PAPER.md, cited as P:<line>) and the readings listed in DESIGN.md.
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import this package. It shares no code with the CUDA path
(`paper_2512_04752_b200/`), and the CUDA path never imports it.

Modules
  tree        ancestor-or-self masks and depths from parent[]
  attention   exact masked tree attention in fp64
  accept      greedy / rejection-sampling tree acceptance (C, via ctypes)
  compact     sequential KV commit of the accepted path
  migrate     model->layer->sample pack / unpack of KV
  strategy    dl, top-n selection, al, t_sd, layer-level search
  realloc     threshold knee and greedy reallocation plan (Eq. 6)

Parity status per function is listed in DESIGN.md ("Oracle pins"); every function here is
pinned by a `-m "not gpu"` test against something other than itself.
"""
