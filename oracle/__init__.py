"""CPU oracle for the NetFuse merged-operator path — TEST INFRASTRUCTURE.

A restatement of the reference's numpy kernels (pkg/src/modelmerge/engine.py)
and of the ops the reference lacks. Used only by tests/, by
__graft_entry__.smoke() as the parity checker, and by bench.py's CPU
baseline / `--impl reference` arm. Never imported by the GPU product path.
Parity pinned against the reference's own outputs (tests/golden/, generated
by oracle/gen_golden.py) for every reference kernel; the extension ops
(GELU, attention, relative attention, padded pools) are unpinned
restatements cross-checked against transformers / torch definitions.
"""
