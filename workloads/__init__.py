"""Seeded, synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no stencil, transfer, smoother,
interpolation or Green's function).  It only produces:

* block layouts (leaf lists ``(level, bi, bj, bk)``) — `layouts`
* analytic source terms sampled at leaf nodes — `sources`
* the five BASELINE.json configurations and small test variants — `configs`

Both `oracle/` and the CUDA path (through `paper_2512_08555_b200`) consume these
arrays; nothing here imports either of them.
"""
