/* generated vector permutation kernel
 * target: x86-avx  width: 512 bits  elem: 8 B  lanes: 8
 * shape (inner-first): (512, 32, 8192)  map (inner-first): (0, 2, 1)
 * shuffle steps: 0  block registers: 1  utilization: 1
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <immintrin.h>
static void vp_adv_0(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 64) { *bs += 8; *bd += 8; return; }
    i[0] = 0; *bs -= 504; *bd -= 504;
    if (++i[1] < 8192) { *bs += 16384; *bd += 512; return; }
    i[1] = 0; *bs -= 134201344; *bd -= 4193792;
    if (++i[2] < 32) { *bs += 512; *bd += 4194304; return; }
    i[2] = 0; *bs -= 15872; *bd -= 130023424;
}
void permute_79c05a3a09aee559(const void *src_v, void *dst_v) {
    const uint32_t *src = (const uint32_t *)src_v;
    uint32_t *dst = (uint32_t *)dst_v;
    { /* loop main: 2097152 iterations, unroll 8 */
        int64_t vp_i[3] = {0, 0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        int64_t s1_s = 0, s1_d = 0;
        int64_t s2_s = 0, s2_d = 0;
        int64_t s3_s = 0, s3_d = 0;
        int64_t s4_s = 0, s4_d = 0;
        int64_t s5_s = 0, s5_d = 0;
        int64_t s6_s = 0, s6_d = 0;
        int64_t s7_s = 0, s7_d = 0;
        __m512i v0, v1, v2, v3, v4, v5, v6, v7;
        for (int64_t vp_it = 0; vp_it < 2097152; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s1_s = vp_bs; s1_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s2_s = vp_bs; s2_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s3_s = vp_bs; s3_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s4_s = vp_bs; s4_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s5_s = vp_bs; s5_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s6_s = vp_bs; s6_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s7_s = vp_bs; s7_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            v0 = _mm512_load_epi32(src + (s0_s + 0) * 2);
            v1 = _mm512_load_epi32(src + (s1_s + 0) * 2);
            v2 = _mm512_load_epi32(src + (s2_s + 0) * 2);
            v3 = _mm512_load_epi32(src + (s3_s + 0) * 2);
            v4 = _mm512_load_epi32(src + (s4_s + 0) * 2);
            v5 = _mm512_load_epi32(src + (s5_s + 0) * 2);
            v6 = _mm512_load_epi32(src + (s6_s + 0) * 2);
            v7 = _mm512_load_epi32(src + (s7_s + 0) * 2);
            _mm512_store_epi32(dst + (s0_d + 0) * 2, v0);
            _mm512_store_epi32(dst + (s1_d + 0) * 2, v1);
            _mm512_store_epi32(dst + (s2_d + 0) * 2, v2);
            _mm512_store_epi32(dst + (s3_d + 0) * 2, v3);
            _mm512_store_epi32(dst + (s4_d + 0) * 2, v4);
            _mm512_store_epi32(dst + (s5_d + 0) * 2, v5);
            _mm512_store_epi32(dst + (s6_d + 0) * 2, v6);
            _mm512_store_epi32(dst + (s7_d + 0) * 2, v7);
        }
    }
}
