/*
 * parl_gpu_debug.h — test hooks of libparl_gpu.so (not part of the drop-in
 * boundary): direct access to the contraction kernel so the tensor-core
 * layouts and fused epilogues can be unit-tested against torch.
 */
#ifndef PARL_GPU_DEBUG_H
#define PARL_GPU_DEBUG_H
#include "parl_gpu.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C[M x N] (epilogue `epi`, see csrc/internal.cuh Epi) = sum_k A(m,k) B(n,k),
 * A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk]; bf16 device operands.
 * path: 0 = tcgen05 (fails with PARL_E_CONFIG if the shape is not supported), 2 = the same without the
 *       trailing device synchronisation (timing loops),
 *       1 = FFMA tile kernel.  Synchronises the current device. */
parl_status parl_debug_gemm_bf16(int path, int M, int N, int K, const void* A, long sam, long sak, const void* B,
                                 long sbn, long sbk, int epi, const float* bias, float* Cf, long ldc,
                                 const float* resid, void* Ca, long ldca, void* Caux, const void* aux_in,
                                 const int32_t* labels, float* part, float* target, void* logits_act,
                                 int n_parts);
/* Shared-prompt attention forward over qkv [T x 3*H*Dh] (bf16, device):
 * out [T x H*Dh] bf16, lse [H x T]; seg/seg_start/seg_end as produced by the
 * packer.  path 0 = tcgen05, 1 = FFMA. */
parl_status parl_debug_attn_bf16(int path, int T, int H, int Dh, int Peff, const int32_t* seg,
                                 const int32_t* seg_start, const int32_t* seg_end, const void* qkv, void* out,
                                 float* lse);
/* Attention backward: dqkv [T x 3*H*Dh] from dout [T x H*Dh], the forward's
 * out and lse; dsum [H x T] is scratch.  path 0 = tcgen05, 1 = FFMA. */
parl_status parl_debug_attn_bwd_bf16(int path, int T, int H, int Dh, int Peff, const int32_t* seg,
                                     const int32_t* seg_start, const int32_t* seg_end, const void* qkv,
                                     const void* out, const void* dout, const float* lse, float* dsum, void* dqkv);
/* Every array K1 wrote for a packed group, concatenated into out (host, int32):
 * tokens, labels, positions, seg, pred [T each], row_ptr [T + 1], scored_pos, scored_label,
 * pred_pos, sample_of, row_idx [S each]  (6T + 1 + 5S entries). */
parl_status parl_debug_group_arrays(parl_group_t g, int32_t* out);
#ifdef __cplusplus
}
#endif
#endif
