/* tw_hpccg_emulation.h -- multi-rank emulation on ONE device (test and
 * proof infrastructure; not part of the reference-facing boundary in
 * tw_hpccg.h, which is what a reference binding includes).
 *
 * P contexts on one GPU act as the z-slab ranks of a multi-GPU run, so the
 * multi-rank algorithm (halo, rank-ordered scalar sums, the NVLink peer
 * protocol, the block-task DAG across ranks) runs -- and is checked against
 * the oracle -- on the single B200 the test pool has.  Kernels that wait on
 * one another never run as separate launches on one device: the group runs
 * the ranks' phases host-sequenced on one stream, or every rank inside ONE
 * launch (the cooperative rank-group kernel; the persistent dispatcher over
 * all ranks' task tables). */
#ifndef TW_HPCCG_EMULATION_H
#define TW_HPCCG_EMULATION_H

#include "tw_hpccg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Emulated rank r of an nranks group on ONE device (no NCCL).  Solvers on
 * such contexts are driven together by tw_cg_group_set_rhs /
 * tw_cg_group_iterate. */
int tw_ctx_init_emulated_rank(tw_ctx* ctx, int rank, int nranks);

/* cgs[r] is rank r's solver (all ranks: the same variant, tile count and
 * dispatch), b[r] its rows of b.  Monolithic: every rank's phases on one
 * stream, loopback copies in place of the NCCL halo and allgathers.  Tasks
 * variant on streams: every rank's DAG nodes phase by phase (halo, SpMV
 * tiles, tile-order / rank-order alpha, x/r tiles, beta_res, p tiles) with
 * the NCCL executor's kernels.  Tasks variant with TW_DISPATCH_PERSISTENT
 * (after tw_cg_group_enable_peer): every rank's task table in ONE
 * dispatcher launch, the cross-rank edges being the peer protocol. */
int tw_cg_group_set_rhs(tw_cg** cgs, int nranks, const double* const* b, int b_is_device);
int tw_cg_group_iterate(tw_cg** cgs, int nranks, int iterations);
/* The group over the NVLink peer transport instead of the loopback copies:
 * the "peers" are the other ranks' buffers on the device (monolithic
 * variant, or the persistent dispatcher). */
int tw_cg_group_enable_peer(tw_cg** cgs, int nranks);
/* The monolithic peer-transport group as ONE cooperative kernel: the ranks'
 * blocks run concurrently and wait on one another's flags (the multi-GPU
 * protocol under real concurrency on one device).  jitter != 0 delays
 * rank-dependent blocks to vary the interleavings.  Synchronous. */
int tw_cg_group_iterate_concurrent(tw_cg** cgs, int nranks, int iterations, int jitter);

#ifdef __cplusplus
}
#endif

#endif /* TW_HPCCG_EMULATION_H */
