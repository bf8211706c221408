/* fs1_shard.h — C ABI of the sharded single-problem FS-1 solve (libfs1.so).
 *
 * One 1D problem too large for one GPU (north_star: "for single
 * problems too large for one GPU, to exchange per-shard scan carries") is split
 * into `world` contiguous segments of whole 256-point tiles, one per rank (GPU).
 * Every K x of Algorithm 1 is the forward and backward
 * recursion of Eq. "recursion" over the whole grid; a segment
 * needs from the others only their totals (forward total at the segment end,
 * backward total at its start: 4 doubles per rank).  So each half-step is
 *
 *     all-gather the ranks' totals of x  ->  fs1_shard_half  ->  totals of y
 *
 * and the caller (the Python driver, paper_2202_10042_b200/shard.py) moves the
 * totals between ranks with one NCCL all-gather per half-step — or lets the kernels
 * move them over peer memory (fused exchange, below) — and owns the loop
 * control (Algorithm 1's while, with the readings of DESIGN.md R2-R6).
 *
 * Supported: ndim 1, FS1_F64, FS1_LOG, batch 1, check_interval >= 1, no warm
 * start.  Arrays are segment slices of the global problem, device pointers,
 * caller-owned; every call is asynchronous on `stream` and never allocates.
 * Totals and partial results are device arrays of doubles (exponents stored as
 * exact doubles).
 */
#ifndef FS1_SHARD_H
#define FS1_SHARD_H

#include "fs1.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fs1_shard_s fs1_shard_t;

/* fs1_shard_plan — plan rank `rank` of `world` for the global problem `desc`.
 *   seg_lo, seg_len : receive this rank's segment [seg_lo, seg_lo + seg_len) of
 *                     the N points (tiles are split as evenly as possible; the
 *                     segment may be empty only if world > tiles: FS1_ERR_ARG).
 *   workspace_bytes : device workspace fs1_shard_* need (256-byte aligned).
 * Errors: FS1_ERR_ARG (world < 1, rank out of range, batch != 1, warm start),
 * FS1_ERR_EPS, FS1_ERR_UNSUPPORTED (dtype/domain/ndim; h/eps (min(n, 256) - 1) > 600, the
 * per-tile fp64 range of DESIGN.md §5.3).                                          */
fs1_status fs1_shard_plan(const fs1_desc* desc, int world, int rank, int device, fs1_shard_t** out,
                          size_t* workspace_bytes, int64_t* seg_lo, int64_t* seg_len);

/* fs1_shard_init — load a, b (segment slices, log-weights if desc.input_is_log),
 * set phi0 = psi0 = 1/N and write phi0's segment totals to tot4
 * (device, 4 doubles).                                                             */
fs1_status fs1_shard_init(const fs1_shard_t* s, const void* a_seg, const void* b_seg, double* tot4,
                          void* workspace, void* stream);

/* fs1_shard_half — one half-step on this segment.
 *   which   : 0 = psi update psi = b ./ (K^T phi),
 *             1 = phi update phi = a ./ (K psi).
 *   hs      : half-step counter (0 for the first psi step; +1 per call that writes).
 *   check   : also compute this rank's part of the marginal error
 *             sum_i |psi_i (K^T phi)_i - b_i| with psi = buffer psi_in.
 *   write   : produce y (0 only for the final check at l = itr_max).
 *   l1      : iteration recorded if y becomes non-finite (l + 1); -1 = use the
 *             plan's device counter (starts at 1, advanced after every phi half-step
 *             called with -1), for replays of a captured CUDA graph.
 *   psi_in, psi_out : psi buffers (0/1): which=0 reads psi_in (check) and writes
 *             psi_out; which=1 reads psi_in.
 *   all_tot : device [world][4] totals of x from every rank (the all-gather).
 *   tot4    : device out, totals of y (write = 1).
 *   errflag : device out [2] = {error partial of this rank, first iteration l1 whose
 *             state became non-finite on this rank (0: none)}.                    */
fs1_status fs1_shard_half(const fs1_shard_t* s, int which, int hs, int check, int write, int l1, int psi_in,
                          int psi_out, const double* all_tot, double* tot4, double* errflag, void* workspace,
                          void* stream);

/* fs1_shard_decide — the loop-top decision of Algorithm 1 line 2 on the
 * device, from every rank's errflag (all_errflag: device [world][2], the all-gather of the
 * fs1_shard_half errflag rows in rank order; the same on every rank):
 *   out4[0] = err = sum of the error partials in rank order,
 *   out4[1] = 0 continue | 1 CONVERGED (tol > 0, err <= tol) | 2 NONFINITE | 4 ITR_MAX (l >= itr_max),
 *   out4[2] = the iteration at the stop (NONFINITE: the smallest non-finite record), out4[3] = 0.
 *   l : the loop-top iteration.  The caller only reads the flag.                     */
fs1_status fs1_shard_decide(const fs1_shard_t* s, const double* all_errflag, int l, double* out4, void* stream);

/* fs1_shard_sum — out[0] = sum over ranks (rank order) of rows[k * stride + col]
 * (device [world][stride]; the cost partials of fs1_shard_finish).                    */
fs1_status fs1_shard_sum(const fs1_shard_t* s, const double* rows, int stride, int col, double* out,
                         void* stream);

/* fs1_shard_cost_totals — Jordan-block pair totals of psi (buffer `psi`) for the
 * return line (R7): device out tot8 = 8 doubles.          */
fs1_status fs1_shard_cost_totals(const fs1_shard_t* s, int psi, double* tot8, void* workspace, void* stream);

/* fs1_shard_finish — this rank's cost partial h sum_k phi_k (W psi)_k over the
 * segment (all_tot8: device [world][8] from fs1_shard_cost_totals), and F = log phi,
 * G = log psi of the segment into u_seg, v_seg (device fp64).  The cost is the sum
 * of the partials over ranks (fixed rank order).  cost_partial may be NULL.        */
fs1_status fs1_shard_finish(const fs1_shard_t* s, int psi, const double* all_tot8, void* u_seg, void* v_seg,
                            double* cost_partial, void* workspace, void* stream);

/* ---- Fused exchange over peer memory.
 * Instead of the caller's all-gather of the totals, the kernels move them: the
 * totals kernel of every production writes this rank's row straight into every
 * rank's mailbox (NVLink peer stores through IPC mappings) and raises a per-rank
 * flag with a system-scope release; the next half-step's kernel acquires the flags
 * and reads the rows from its own mailbox.  No host step, no collective launch.
 *
 * fs1_shard_mailbox_bytes — size of one rank's mailbox for `world` ranks
 *   (world <= FS1_SHARD_MAXW = 16).
 * fs1_shard_mailbox_alloc — cudaMalloc + zero a mailbox on `device` and return its
 *   CUDA IPC handle (64 bytes into ipc_handle, may be NULL).  One mailbox per rank per
 *   solve: its flags and epoch must start at zero.
 * fs1_shard_mailbox_open / _close — map / unmap a peer's mailbox from its IPC handle
 *   (another process; a rank's own mailbox or one in this process is used directly).
 * fs1_shard_mailbox_free — free a mailbox from fs1_shard_mailbox_alloc.
 * fs1_shard_set_mailboxes — boxes[world]: every rank's mailbox as seen from this
 *   rank's device (boxes[rank] = its own); NULL switches back to the all_tot path.
 *   With mailboxes set, fs1_shard_init and fs1_shard_half (write = 1) deliver the
 *   totals themselves and fs1_shard_half ignores all_tot (may be NULL); tot4 still
 *   receives this rank's totals.  All ranks must issue the same sequence of calls.
 * Errors: FS1_ERR_ARG (world out of range, NULL pointers), FS1_ERR_CUDA.            */
size_t fs1_shard_mailbox_bytes(int world);
fs1_status fs1_shard_mailbox_alloc(int world, int device, void** box, void* ipc_handle);
fs1_status fs1_shard_mailbox_open(const void* ipc_handle, int device, void** box);
fs1_status fs1_shard_mailbox_close(void* box);
fs1_status fs1_shard_mailbox_free(void* box);
fs1_status fs1_shard_set_mailboxes(fs1_shard_t* s, void* const* boxes);

void fs1_shard_destroy(fs1_shard_t* s);

#ifdef __cplusplus
}
#endif
#endif /* FS1_SHARD_H */
