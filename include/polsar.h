/*
 * polsar.h -- C-ABI of the B200 (sm_100a) hot path of arXiv 1807.08084:
 * batched inverse and determinant of 3x3 Hermitian positive-definite PolSAR
 * multilook covariance matrices, plus the search-window distance kernel.
 *
 * Library: paper_1807_08084_b200/libpolsar.so (nvcc, -gencode
 * arch=compute_100a,code=sm_100a).  No torch types cross this boundary: plain
 * pointers, sizes, an int dtype code and a cudaStream_t passed as void*.
 *
 * ---------------------------------------------------------------------------
 * Data layout (all entry points)
 *   Packed Hermitian Z = [[a, b, c], [conj b, d, e], [conj c, conj e, f]],
 *   a, d, f real, b, c, e complex; only the upper triangle is stored
 *   (PAPER.md:136-153 [§II-A], 456-457 [§III-A]).  Planar structure of
 *   arrays: plane k of a buffer starts at element k*ld, pixel p of plane k is
 *   element k*ld + p.
 *     input  z   : 9 planes   0 a, 1 Re b, 2 Im b, 3 Re c, 4 Im c, 5 d,
 *                             6 Re e, 7 Im e, 8 f
 *     output out : 11 planes  0..8 the upper triangle of Z^-1 in the same
 *                             field order (a_i, b_i, c_i, d_i, e_i, f_i),
 *                             9 det Z, 10 det Z^-1 (= t of Alg. 2)
 *     status     : n bytes (nullable): 0 OK, 1 SINGULAR, 2 NOT_PD
 *   Element type by `dtype`:
 *     POLSAR_F32        fp32 storage, fp64 arithmetic, each output rounded
 *                       once to fp32 (the accurate default; R-11)
 *     POLSAR_F64        fp64 storage, fp64 arithmetic with every cofactor
 *                       evaluated to ~2u (FMA two-products, one exact sum)
 *                       and a compensated Eq. 6 determinant: relative error
 *                       ~ kappa u (<= 1e-12 at kappa <= 1e4; R-16)
 *     POLSAR_F32_PLAIN  fp32 storage and arithmetic, Alg. 2 as printed
 *     POLSAR_F64_PLAIN  fp64 storage and arithmetic, Alg. 2 as printed
 *     POLSAR_F64_EFT    fp64 storage, error-free evaluation of Alg. 2 (the
 *                       determinant's cofactors carried as hi + lo): a few
 *                       ulp at any kappa, ~1.5x the FP64 work of POLSAR_F64
 *                       (polsar_inv_det, polsar_inv_det_blocks and
 *                       polsar_inv_det_host only; elsewhere POLSAR_ENOTSUP)
 *   The 128-bit vector path is taken when every plane base is 16-byte
 *   aligned and ld is a multiple of 16/sizeof(element); otherwise a scalar
 *   path runs the same device function and yields identical bits.
 *
 * Ownership and conventions
 *   The caller owns every buffer (device memory, e.g. from torch).  The
 *   library never allocates device memory, frees or (except
 *   polsar_inv_det_host) synchronises; kernels are enqueued on
 *   `cuda_stream` (NULL = legacy default stream) and return immediately.
 *   Host-side argument checks are synchronous; asynchronous device faults
 *   surface at the caller's next synchronisation.  n == 0 is a successful
 *   no-op.  Stateless and thread-safe.  Non-OK pixels still receive whatever
 *   the arithmetic yields (possibly inf/nan): mask by status.
 *   No fast-math: division, reciprocal and sqrt are IEEE round-to-nearest
 *   (PAPER.md:631-640 [§III-C]).
 *
 * Return codes: POLSAR_OK, POLSAR_EINVAL (null pointer, n < 0, ld < n, bad
 * dtype / radius / range), POLSAR_ECUDA (launch error), POLSAR_ENOTSUP.
 * polsar_last_error() returns a static string describing the last failure
 * on the calling thread.
 */
#ifndef POLSAR_H
#define POLSAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    POLSAR_F32 = 0,
    POLSAR_F64 = 1,
    POLSAR_F32_PLAIN = 2,
    POLSAR_F64_PLAIN = 3,
    POLSAR_F64_EFT = 4
} polsar_dtype;

enum { POLSAR_OK = 0, POLSAR_EINVAL = 1, POLSAR_ECUDA = 2, POLSAR_ENOTSUP = 3 };
enum { POLSAR_STATUS_OK = 0, POLSAR_STATUS_SINGULAR = 1, POLSAR_STATUS_NOT_PD = 2 };

/* polsar_inv_det -- the paper's reduced-arithmetic closed form, Alg. 2
 * (PAPER.md:480-545 [§III-A, Alg. 2]; Eq. (3) cofactors PAPER.md:168-189,
 * Eq. (4) A^-1 = adj(A)/det A PAPER.md:390-397, Eq. (6) real-part determinant
 * PAPER.md:411-445).  One thread per matrix group, HBM-streaming.
 *   z      : device, 9 planes of n elements, plane stride ld
 *   out    : device, 11 planes of n elements, plane stride ld (same ld)
 *   status : device, n bytes or NULL.  SINGULAR iff !(det > tau*a*d*f) or a
 *            result is non-finite, tau = 16 u_in (u_in = 2^-24 for fp32
 *            storage, 2^-53 for fp64): the full-rank check of PAPER.md:469-476
 *            read as a scaled threshold (R-5).
 *   n      : pixel count (>= 0);  ld >= n. */
int polsar_inv_det(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                   int dtype, void* cuda_stream);

/* polsar_inv_det_cholesky -- the comparison method, Alg. 1 (PAPER.md:279-378
 * [§II-B, Alg. 1]) with the conjugation of l21 corrected to
 * l21 = (conj(e) - l20 conj(l10)) v1 (R-1; the printed line,
 * PAPER.md:298, is wrong) and det Z^-1 = (v0 v1 v2)^2 (R-14).  Same layout,
 * ownership and errors as polsar_inv_det; status NOT_PD iff a radicand of
 * step 1 is <= 0 or non-finite, else SINGULAR by the same threshold rule. */
int polsar_inv_det_cholesky(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                            int dtype, void* cuda_stream);

/* polsar_inv_det_blocks -- multi-frequency PolSAR pixels whose covariance is
 * block diagonal with nblocks Hermitian 3x3 blocks, one per frequency band
 * (PAPER.md:1043-1055 [§V]): Alg. 2 on each block.
 *   z      : device, 9*nblocks planes (block b at planes 9b..9b+8, field order
 *            as above), plane stride ld
 *   out    : device, 9*nblocks + 2 planes: block inverses at 9b..9b+8, then
 *            det and det^-1 of the whole block-diagonal matrix (products of
 *            the block values in the arithmetic type, rounded once)
 *   status : device, n bytes or NULL: the worst block status
 *   nblocks: 1..64;  dtype, ownership and errors as polsar_inv_det. */
int polsar_inv_det_blocks(const void* z, void* out, uint8_t* status, int64_t n, int64_t ld,
                          int nblocks, int dtype, void* cuda_stream);

/* polsar_window_workspace_bytes -- bytes of device workspace the window
 * entry points (polsar_window_distance, polsar_nlm_filter, polsar_window_kl)
 * need for a slab of slab_rows x width pixels at this radius and dtype: the
 * largest need of the three.  (polsar_nlm_filter stores the 2R(R+1) forward
 * pair weights of the pixels of one band of 1024 output rows plus its 2R
 * halo rows, ~1.07 KB per band pixel at R = 11 with fp32 weights -- 2.3 GB
 * for a 2048-pixel-wide slab of any height; the window and KL kernels need
 * ~40 B per slab pixel.) */
size_t polsar_window_workspace_bytes(int64_t slab_rows, int64_t width, int radius, int dtype);

/* polsar_window_workspace_bytes_for -- the same for one entry point:
 * entry 0 polsar_window_distance, 1 polsar_nlm_filter, 2 polsar_window_kl
 * (0 for an invalid entry, negative or > 2^40-pixel sizes, or an
 * unsupported dtype / radius).  It is the need of the kernel form that entry
 * point runs for (dtype, radius) -- fixed at compile time, independent of the
 * environment -- so a workspace of this size serves every call of that entry
 * point with these sizes.  A UAVSAR-scale slab (10000 x 40000 pixels) needs
 * ~16 GB for the window and KL sums and ~46 GB for the NLM (one band). */
size_t polsar_window_workspace_bytes_for(int entry, int64_t slab_rows, int64_t width, int radius,
                                         int dtype);

/* polsar_window_distance -- non-local-means search-window sum (the workload
 * of PAPER.md:77-80 [§I]; formula of BASELINE.json configs[4]):
 *   W_i = sum_{j in N(i)} exp(-d_ij / h),
 *   d_ij = L [ln det((Z_i + Z_j)/2) - (ln det Z_i + ln det Z_j)/2],
 * N(i) the (2R+1)x(2R+1) window centred on i clipped to the image (R-12).
 *   z         : device, 9 planes of a slab of slab_rows x width pixels
 *               (row-major, slab_rows*width <= 2^40, else EINVAL), plane
 *               stride ld >= slab_rows*width.  The slab is
 *               exactly the in-image rows around the output rows, so clipping
 *               at the slab edge equals clipping at the image edge.
 *   out_row_begin, out_row_end : slab rows whose W is written (0 <= b <= e
 *               <= slab_rows); out receives (e - b) x width values, row-major.
 *   radius R (>= 0, <= 16; the paper's 23x23 window is R = 11), looks L (> 0),
 *               h (> 0).
 *   workspace : device, polsar_window_workspace_bytes_for(0, slab_rows, width, radius, dtype)
 *               (or the all-entry-points polsar_window_workspace_bytes)
 *   dtype     : POLSAR_F32 (fp32 storage, fp64 pair determinant, fp32
 *               weight) or POLSAR_F64 (fp64 throughout), or the _PLAIN
 *               variants (storage precision throughout).
 * Pixels must be Hermitian positive definite: a pixel whose determinant is
 * not positive or not finite makes W NaN on every pixel whose window holds it
 * (likewise for polsar_window_kl and both outputs of polsar_nlm_filter).
 * Results are bit-reproducible: any slab decomposition gives the same bits. */
int polsar_window_distance(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                           int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                           double h, void* workspace, void* out, int dtype, void* cuda_stream);

/* polsar_window_kl -- the same window sum with the symmetric Wishart
 * Kullback-Leibler distance (one of the divergences that need Z^-1, PAPER.md:
 * 70-76 [§I]):
 *   d_ij = L [ (tr(Z_i^-1 Z_j) + tr(Z_j^-1 Z_i)) / 2 - 3 ],  W_i = sum_j exp(-d_ij / h).
 * Z^-1 of every slab pixel comes from Alg. 2 (K1's device function); each
 * pair is then two 9-term trace products in fp64 (as one 20-term product on
 * the FP64 tensor cores).  Arguments,
 * workspace (polsar_window_workspace_bytes_for(2, ...)) and errors as
 * polsar_window_distance; radius <= 12; dtype POLSAR_F32 or POLSAR_F64
 * (POLSAR_F32_PLAIN returns ENOTSUP). */
int polsar_window_kl(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                     int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                     double h, void* workspace, void* out, int dtype, void* cuda_stream);

/* polsar_nlm_filter -- non-local-means filter output with the same search-
 * window weights (the NLM filter with stochastic distances of PAPER.md:77-80
 * [§I]); for 1 <= R <= 12 the symmetric pass stores each
 * forward weight once and a gather pass forms Zhat, band by band (1024 output
 * rows per band, each with its own R-row halos; the bands give the same bits
 * as one pass over the slab would):
 *   W_i = sum_j exp(-d_ij / h),   Zhat_i = sum_j exp(-d_ij / h) Z_j / W_i.
 * Arguments as polsar_window_distance, plus
 *   out_w  : device, (e - b) x width values of W, or NULL
 *   out_z  : device, 9 planes of (e - b) x width filtered pixels (packed
 *            field order), plane stride ld_out >= (e - b) * width.
 * Workspace: polsar_window_workspace_bytes_for(1, slab_rows, width, radius, dtype). */
int polsar_nlm_filter(const void* z, int64_t ld, int64_t width, int64_t slab_rows,
                      int64_t out_row_begin, int64_t out_row_end, int radius, double looks,
                      double h, void* workspace, void* out_w, void* out_z, int64_t ld_out,
                      int dtype, void* cuda_stream);

/* polsar_checksum -- verification reduction (support for multi-GPU
 * bit-identity).  Adds to result[0] (uint64, wrapping)
 * sum_p sum_k mix64(bits(plane k, pixel p) ^ key(pix_offset + p, k)) over
 * nplanes planes of n elements (stride ld, element size 4 or 8 bytes by
 * dtype), and, if status != NULL, adds the counts of status 0/1/2 to
 * result[1..3].  Order-independent, so per-rank results summed over ranks
 * equal the single-GPU result bit for bit.  result: device, 4 x uint64. */
int polsar_checksum(const void* planes, int64_t n, int64_t ld, int nplanes, int dtype,
                    int64_t pix_offset, const uint8_t* status, uint64_t* result,
                    void* cuda_stream);

/* polsar_inv_det_host -- end-to-end entry point on HOST buffers (pinned for
 * full speed).  Streams the batch through caller-provided device staging
 * buffers in chunks, three slots deep: the H2D copy of chunk k+1, the kernel
 * on chunk k and the D2H copy of chunk k-1 overlap on three caller streams
 * (the out-of-core path of PAPER.md:947-963 [§IV-C]).  algo 0 = Alg. 2,
 * 1 = Alg. 1.
 *   z_host   : 9 planes of n elements, plane stride ld_host
 *   out_host : 11 planes, stride ld_host;  status_host : n bytes or NULL
 *   dev_ws   : device workspace of ws_bytes; the chunk size is derived from it
 *              (polsar_host_chunk_pixels; 256-byte aligned pointer required).
 *   stream_h2d, stream_compute, stream_d2h : three distinct CUDA streams.
 * Host planes whose stride ld_host * element size exceeds the device's
 * cudaDevAttrMaxPitch (2^31 - 1 B) are copied plane by plane instead of by
 * one 2D copy per chunk.  Pageable host memory works, at pageable speed.
 * Synchronous: returns after the last D2H copy has completed; on every path,
 * error paths included, it first synchronises all three streams, so nothing
 * it enqueued still touches the host buffers or dev_ws (the only entry point
 * that synchronises). */
int polsar_inv_det_host(const void* z_host, void* out_host, uint8_t* status_host, int64_t n,
                        int64_t ld_host, int dtype, int algo, void* dev_ws, size_t ws_bytes,
                        void* stream_h2d, void* stream_compute, void* stream_d2h);

/* pixels per chunk polsar_inv_det_host uses for a workspace of ws_bytes */
int64_t polsar_host_chunk_pixels(size_t ws_bytes, int dtype);

/* static description of the last error on this thread ("" if none) */
const char* polsar_last_error(void);

/* library version, e.g. 0x000100 */
int polsar_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POLSAR_H */
