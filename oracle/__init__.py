"""CPU fp64 ORACLE for the multi-dimensional tensor-parallel linear layer.

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import anything here.
The product path (`paper_2110_14883_b200`, the C-ABI library) never imports,
links or executes this package, and this package never imports the product.
The two share no code; the only common module is `synth` (seeded inputs, no
method arithmetic).

What it computes (PAPER.md = P:Lnnn, SPEC.md = S:Lnnn):

  dense.py     Y = alpha*X*W + b, dX = alpha*dY*W^T, dW = alpha*X^T*dY, db = 1^T dY
               in fp64 - the plain definition every TP mode re-associates
               (S:L198-206).
  grid.py      grids and per-axis groups.
  shards.py    per-rank block extents for X, W, Y, bias in every mode
               (P:L524 2D, P:L526 2.5D, P:L528 3D, P:L486-488 1D).
  fabric.py    simulated collectives on per-rank fp64 buffers with the element
               ledger of SPEC's conventions.
  programs.py  explicit rank-by-rank fwd/bwd programs of 1D col/row, 2D SUMMA,
               2.5D and 3D, following SURVEY.md section 8(a) rows a-3 .. a-10.
  closed_forms.py  Table tp-comm-vol verbatim, our schedule's
               counted volumes, per-rank memory closed forms.
  sampled.py   entries of full-size outputs computed one by one (bench-size
               parity).

Pins (what fixes this oracle to something other than itself) live in
tests/test_oracle_*.py; see DESIGN.md "Oracle pins". Parity status per function:
all functions are pinned, except the absolute allocator peak bytes of the
paper's memory test, which are "parity unpinned" (only ratios are compared).
"""
