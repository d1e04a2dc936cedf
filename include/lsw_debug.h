/*
 * lsw_debug.h -- tuning hooks of liblsw.so.  Not part of the hot path and not
 * needed by users; they expose measurement state that the kernels record only
 * when enabled by environment variables read at lsw_create:
 *
 *   LSW_TC_TRACE=1   the tensor-core switch kernel stamps %globaltimer (ns) at
 *                    16 pipeline event slots of its first 2048 tiles in 4 CTAs
 *                    spread over the grid (layout [cta][tile][event], events in
 *                    switch_tc.cu EV_*: W issued, A issued, A full, MMA start,
 *                    MMA done, epilogue saw W, epilogue saw accumulators, stage
 *                    freed, epilogue done, MMA got a free accumulator buffer,
 *                    MMAs issued, first sub-tile done, A production began, A
 *                    ring slot free); 0 = not reached.
 */
#ifndef LSW_DEBUG_H_
#define LSW_DEBUG_H_

#include "lsw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Copy up to n uint64 trace words of the last switch launch into host_out (host
 * memory).  Returns the number copied in *n_out (0 when tracing is off or the
 * ctx uses the SIMT switch).  Synchronizes the device.  LSW_E_ARG on null. */
LSW_API lsw_status lsw_debug_switch_trace(lsw_ctx* ctx, uint64_t* host_out, int64_t n, int64_t* n_out);

/* Launch-count ablation (the paper's "simple merge" row of
 * Tab. 6): the Eq. 6 merge of lsw_merge_all_layers, but ONE launch
 * of the same tensor-core kernel per adapted matrix (7 x L launches, each over
 * that matrix's tiles).  Same result (bitwise) as the single launch.  State
 * must be `none` (LSW_E_STATE otherwise) and becomes merged(idx, gate);
 * LSW_E_UNSUPPORTED for the SIMT switch.  Enqueue-only (graph-capturable). */
LSW_API lsw_status lsw_debug_merge_per_matrix(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSW_DEBUG_H_ */
