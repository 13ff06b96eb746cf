"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no aggregation, packing,
sharding, encoder math, pooling).  It only *defines the inputs*:

* ``synth.configs``  -- encoder shapes and workload recipes;
* ``synth.workload`` -- partition sizes, text lengths and token ids;
* ``synth.weights``  -- random-init encoder weights rounded to bf16, and the flat
  weight-blob layout documented in ``include/surge.h``.

Both ``oracle/`` and ``paper_2605_01060_b200`` may import it; it imports neither.
"""
