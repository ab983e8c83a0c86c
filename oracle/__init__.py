"""oracle/ -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A CPU restatement of the Faster-MoA agent-execution hot path (reference
``/root/reference/proj/core``) used only as the *checker* for the B200 path:

* ``rng``        -- splitmix64 / fnv1a / RngStream          (rng.hpp:14-103)
* ``topology``   -- Topology::tree/tree_custom/all_to_all   (topology.cpp:43-196)
* ``prompt``     -- PromptTemplate / assemble / without     (prompt.cpp:8-118)
* ``router``     -- SlotPlan slot-filling state machine     (router.cpp:9-184)
* ``metricq``    -- Algorithm 1 + MockProvider              (metricq.cpp:10-194, embedding.cpp:86-120)
* ``model``      -- CPU transformer agent (numpy fp32 over the same bf16 weights;
                    no reference implementation exists -> parity of logits/tokens
                    is pinned only against this restatement)
* ``engine``     -- the tick engine protocol (pdsim.cpp:155-418 semantics on ticks)
* ``orchestrator`` -- run_query + EE gate + summarize       (orchestrator.cpp:130-382)

Pinning: rng/topology/prompt/router/metricq are checked against the reference
itself (oracle/_ref/libmoaref.so, built by oracle/ref/Makefile from the
reference sources) and against golden vectors transcribed from the
reference's own tests (tests/golden/).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference arm may import this package.
"""
