"""ORACLE -- test infrastructure only.  NOT part of the product path.

A plain, slow, obviously-correct CPU implementation of what libsurge computes,
written from the paper (arxiv 2605.01060, /root/reference/PAPER.md, cited "P:n")
and the north star (BASELINE.json).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import,
call or execute anything under ``oracle/``.  It shares no code with the CUDA path
(``paper_2605_01060_b200``) and neither imports the other; the only common module
is ``synth`` (seeded input generators, no method arithmetic).

Modules
-------
``oracle.aggregator`` -- Alg.1 AddPartition/Flush with the Lemma
     and Theorem invariants; packing of a SuperBatch into
    cu_seqlens / partition offset tables; the LPT shard plan (north star).
``oracle.encoder`` -- fp64 BERT-class encoder applied to each text independently,
    masked mean-pool and L2 normalisation ("384-dimensional L2-normalized
    embeddings"; architecture from the public BERT definition the north star names).
``oracle.pipeline`` -- the end-to-end plain definition: partitions in, per-partition
    embedding matrices out (P:165 problem statement), via the aggregator.

Precision: fp64 throughout (the paper does not fix precision; the task rule is
fp64 unless it does -- see DESIGN.md "Readings").

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): transformers BertModel fp64
(independent library routine), closed forms for pooling and LayerNorm, brute-force
and special-case attention, SPEC/paper worked examples for the aggregator
(tests/golden/paper_values.json), Monte-Carlo fill ratio vs eq:fill-ratio,
adversarial Lemma orders, LPT brute-force re-check.  Functions without an
independent pin are marked "parity unpinned" in their docstring and in DESIGN.md.
"""
