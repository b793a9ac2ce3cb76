/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the GPU permutation path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product path
 * (paper_2506_03686_b200/) never links or calls it.
 *
 * Plain-C restatement of the reference's scalar oracle:
 *   naive_permute            /root/reference/pkg/src/vecperm/core.py:192-204
 *   ElementBijection.__call__ /root/reference/pkg/src/vecperm/core.py:173-178
 *   permuted_layout           /root/reference/pkg/src/vecperm/core.py:128-132
 *   compute_strides           /root/reference/pkg/src/vecperm/core.py:44-55
 *
 * Conventions follow core.py:1-7: dims are innermost-first, sigma[j] is the
 * source dim that lands at destination position j (inner-first).  The
 * bijection is out[i] = in[f(i)] with
 *   f(i) = sum_j digit_j(i; out.dims) * in.strides[sigma[j]].
 * Elements are opaque words of elem_bytes bytes (core.py:29,36-41 accepts
 * 4 and 8; this restatement accepts any width, which the tests use for the
 * 1/2/16-byte superset).
 *
 * Parity pin: tests/test_oracle.py checks this file against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 *
 * The destination walk uses an incremental mixed-radix counter (the same
 * digits as core.py:176-177, advanced instead of re-divided) and is split
 * across OpenMP threads by destination range; each thread seeds its counter
 * with the closed-form digits of its first offset.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define VPO_MAX_RANK 128

/* return codes mirror LayoutError cases of core.py */
enum { VPO_OK = 0, VPO_EINVAL = 1 };

static int check_args(int rank, const int64_t *dims, const int32_t *sigma, int elem_bytes)
{
    if (rank < 1 || rank > VPO_MAX_RANK) return VPO_EINVAL;      /* core.py:46-47 */
    if (elem_bytes < 1 || elem_bytes > 64) return VPO_EINVAL;
    unsigned char seen[VPO_MAX_RANK];
    memset(seen, 0, sizeof seen);
    for (int k = 0; k < rank; ++k) {
        if (dims[k] < 1) return VPO_EINVAL;                          /* core.py:50-54 */
        if (sigma[k] < 0 || sigma[k] >= rank || seen[sigma[k]]) return VPO_EINVAL; /* core.py:100-101 */
        seen[sigma[k]] = 1;
    }
    return VPO_OK;
}

int vpo_num_elements(int rank, const int64_t *dims, int64_t *n_out)
{
    int64_t n = 1;
    for (int k = 0; k < rank; ++k) n *= dims[k];
    *n_out = n;
    return VPO_OK;
}

/* f(i) for a batch of destination offsets (ElementBijection.__call__). */
int vpo_bijection(int rank, const int64_t *dims, const int32_t *sigma,
                  const int64_t *dst_offsets, int64_t count, int64_t *src_offsets)
{
    if (check_args(rank, dims, sigma, 4) != VPO_OK) return VPO_EINVAL;
    int64_t in_strides[VPO_MAX_RANK], out_dims[VPO_MAX_RANK], out_strides[VPO_MAX_RANK],
        src_of_pos[VPO_MAX_RANK];
    in_strides[0] = 1;
    for (int k = 1; k < rank; ++k) in_strides[k] = in_strides[k - 1] * dims[k - 1];
    for (int j = 0; j < rank; ++j) {
        out_dims[j] = dims[sigma[j]];
        src_of_pos[j] = in_strides[sigma[j]];
    }
    out_strides[0] = 1;
    for (int j = 1; j < rank; ++j) out_strides[j] = out_strides[j - 1] * out_dims[j - 1];
    for (int64_t t = 0; t < count; ++t) {
        int64_t i = dst_offsets[t], s = 0;
        for (int j = 0; j < rank; ++j) s += ((i / out_strides[j]) % out_dims[j]) * src_of_pos[j];
        src_offsets[t] = s;
    }
    return VPO_OK;
}

/* out[i] = in[f(i)] over the whole tensor (naive_permute). */
int vpo_naive_permute(int rank, const int64_t *dims, const int32_t *sigma, int elem_bytes,
                      const void *src_v, void *dst_v, int num_threads)
{
    if (check_args(rank, dims, sigma, elem_bytes) != VPO_OK) return VPO_EINVAL;
    const unsigned char *src = (const unsigned char *)src_v;
    unsigned char *dst = (unsigned char *)dst_v;
    int64_t in_strides[VPO_MAX_RANK], out_dims[VPO_MAX_RANK], step[VPO_MAX_RANK];
    in_strides[0] = 1;
    for (int k = 1; k < rank; ++k) in_strides[k] = in_strides[k - 1] * dims[k - 1];
    int64_t n = 1;
    for (int j = 0; j < rank; ++j) {
        out_dims[j] = dims[sigma[j]];
        step[j] = in_strides[sigma[j]];
        n *= out_dims[j];
    }
    const int eb = elem_bytes;
#ifdef _OPENMP
    if (num_threads < 1) num_threads = omp_get_max_threads();
    if (n < (1 << 16)) num_threads = 1;
#pragma omp parallel num_threads(num_threads)
#endif
    {
        int nt = 1, tid = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        tid = omp_get_thread_num();
#endif
        int64_t lo = n * tid / nt, hi = n * (tid + 1) / nt;
        if (lo < hi) {
            int64_t digit[VPO_MAX_RANK];
            int64_t rem = lo, s = 0;
            for (int j = 0; j < rank; ++j) {           /* closed form, core.py:176-177 */
                digit[j] = rem % out_dims[j];
                rem /= out_dims[j];
                s += digit[j] * step[j];
            }
            for (int64_t i = lo; i < hi; ++i) {
                switch (eb) {
                case 4: ((uint32_t *)dst)[i] = ((const uint32_t *)src)[s]; break;
                case 8: ((uint64_t *)dst)[i] = ((const uint64_t *)src)[s]; break;
                default: memcpy(dst + i * eb, src + s * eb, (size_t)eb); break;
                }
                for (int j = 0; j < rank; ++j) {       /* advance the destination digits */
                    s += step[j];
                    if (++digit[j] < out_dims[j]) break;
                    s -= step[j] * out_dims[j];
                    digit[j] = 0;
                }
            }
        }
    }
    return VPO_OK;
}
