/* generated vector permutation kernel
 * target: x86-avx  width: 512 bits  elem: 4 B  lanes: 16
 * shape (inner-first): (4096, 4096)  map (inner-first): (1, 0)
 * shuffle steps: 4  block registers: 16  utilization: 1
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <immintrin.h>
static const uint32_t vp_tab0[16] = {0, 16, 2, 18, 4, 20, 6, 22, 8, 24, 10, 26, 12, 28, 14, 30};
static const uint32_t vp_tab1[16] = {1, 17, 3, 19, 5, 21, 7, 23, 9, 25, 11, 27, 13, 29, 15, 31};
static const uint32_t vp_tab2[16] = {0, 1, 16, 17, 4, 5, 20, 21, 8, 9, 24, 25, 12, 13, 28, 29};
static const uint32_t vp_tab3[16] = {2, 3, 18, 19, 6, 7, 22, 23, 10, 11, 26, 27, 14, 15, 30, 31};
static const uint32_t vp_tab4[16] = {0, 1, 2, 3, 16, 17, 18, 19, 8, 9, 10, 11, 24, 25, 26, 27};
static const uint32_t vp_tab5[16] = {4, 5, 6, 7, 20, 21, 22, 23, 12, 13, 14, 15, 28, 29, 30, 31};
static const uint32_t vp_tab6[16] = {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23};
static const uint32_t vp_tab7[16] = {8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31};
static void vp_adv_0(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 256) { *bs += 65536; *bd += 16; return; }
    i[0] = 0; *bs -= 16711680; *bd -= 4080;
    if (++i[1] < 256) { *bs += 16; *bd += 65536; return; }
    i[1] = 0; *bs -= 4080; *bd -= 16711680;
}
void permute_fb8dfee3288b9468(const void *src_v, void *dst_v) {
    const uint32_t *src = (const uint32_t *)src_v;
    uint32_t *dst = (uint32_t *)dst_v;
    const __m512i t0 = _mm512_loadu_epi32(vp_tab0);
    const __m512i t1 = _mm512_loadu_epi32(vp_tab1);
    const __m512i t2 = _mm512_loadu_epi32(vp_tab2);
    const __m512i t3 = _mm512_loadu_epi32(vp_tab3);
    const __m512i t4 = _mm512_loadu_epi32(vp_tab4);
    const __m512i t5 = _mm512_loadu_epi32(vp_tab5);
    const __m512i t6 = _mm512_loadu_epi32(vp_tab6);
    const __m512i t7 = _mm512_loadu_epi32(vp_tab7);
    { /* loop main: 65536 iterations, unroll 1 */
        int64_t vp_i[2] = {0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        __m512i v0, v1, v2, v3, v4, v5, v6, v7, v8, v9, v10, v11, v12, v13, v14, v15, v16, v17;
        for (int64_t vp_it = 0; vp_it < 65536; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            v0 = _mm512_load_epi32(src + s0_s + 0);
            v1 = _mm512_load_epi32(src + s0_s + 4096);
            v2 = _mm512_load_epi32(src + s0_s + 8192);
            v3 = _mm512_load_epi32(src + s0_s + 12288);
            v4 = _mm512_load_epi32(src + s0_s + 16384);
            v5 = _mm512_load_epi32(src + s0_s + 20480);
            v6 = _mm512_load_epi32(src + s0_s + 24576);
            v7 = _mm512_load_epi32(src + s0_s + 28672);
            v8 = _mm512_load_epi32(src + s0_s + 32768);
            v9 = _mm512_load_epi32(src + s0_s + 36864);
            v10 = _mm512_load_epi32(src + s0_s + 40960);
            v11 = _mm512_load_epi32(src + s0_s + 45056);
            v12 = _mm512_load_epi32(src + s0_s + 49152);
            v13 = _mm512_load_epi32(src + s0_s + 53248);
            v14 = _mm512_load_epi32(src + s0_s + 57344);
            v15 = _mm512_load_epi32(src + s0_s + 61440);
            v16 = _mm512_permutex2var_epi32(v0, t0, v1);
            v17 = _mm512_permutex2var_epi32(v0, t1, v1);
            v0 = _mm512_permutex2var_epi32(v2, t0, v3);
            v1 = _mm512_permutex2var_epi32(v2, t1, v3);
            v2 = _mm512_permutex2var_epi32(v4, t0, v5);
            v3 = _mm512_permutex2var_epi32(v4, t1, v5);
            v4 = _mm512_permutex2var_epi32(v6, t0, v7);
            v5 = _mm512_permutex2var_epi32(v6, t1, v7);
            v6 = _mm512_permutex2var_epi32(v8, t0, v9);
            v7 = _mm512_permutex2var_epi32(v8, t1, v9);
            v8 = _mm512_permutex2var_epi32(v10, t0, v11);
            v9 = _mm512_permutex2var_epi32(v10, t1, v11);
            v10 = _mm512_permutex2var_epi32(v12, t0, v13);
            v11 = _mm512_permutex2var_epi32(v12, t1, v13);
            v12 = _mm512_permutex2var_epi32(v14, t0, v15);
            v13 = _mm512_permutex2var_epi32(v14, t1, v15);
            v14 = _mm512_permutex2var_epi32(v16, t2, v0);
            v15 = _mm512_permutex2var_epi32(v16, t3, v0);
            v0 = _mm512_permutex2var_epi32(v17, t2, v1);
            v16 = _mm512_permutex2var_epi32(v17, t3, v1);
            v1 = _mm512_permutex2var_epi32(v2, t2, v4);
            v17 = _mm512_permutex2var_epi32(v2, t3, v4);
            v2 = _mm512_permutex2var_epi32(v3, t2, v5);
            v4 = _mm512_permutex2var_epi32(v3, t3, v5);
            v3 = _mm512_permutex2var_epi32(v6, t2, v8);
            v5 = _mm512_permutex2var_epi32(v6, t3, v8);
            v6 = _mm512_permutex2var_epi32(v7, t2, v9);
            v8 = _mm512_permutex2var_epi32(v7, t3, v9);
            v7 = _mm512_permutex2var_epi32(v10, t2, v12);
            v9 = _mm512_permutex2var_epi32(v10, t3, v12);
            v10 = _mm512_permutex2var_epi32(v11, t2, v13);
            v12 = _mm512_permutex2var_epi32(v11, t3, v13);
            v11 = _mm512_permutex2var_epi32(v14, t4, v1);
            v13 = _mm512_permutex2var_epi32(v14, t5, v1);
            v1 = _mm512_permutex2var_epi32(v15, t4, v17);
            v14 = _mm512_permutex2var_epi32(v15, t5, v17);
            v15 = _mm512_permutex2var_epi32(v0, t4, v2);
            v17 = _mm512_permutex2var_epi32(v0, t5, v2);
            v0 = _mm512_permutex2var_epi32(v16, t4, v4);
            v2 = _mm512_permutex2var_epi32(v16, t5, v4);
            v4 = _mm512_permutex2var_epi32(v3, t4, v7);
            v16 = _mm512_permutex2var_epi32(v3, t5, v7);
            v3 = _mm512_permutex2var_epi32(v5, t4, v9);
            v7 = _mm512_permutex2var_epi32(v5, t5, v9);
            v5 = _mm512_permutex2var_epi32(v6, t4, v10);
            v9 = _mm512_permutex2var_epi32(v6, t5, v10);
            v6 = _mm512_permutex2var_epi32(v8, t4, v12);
            v10 = _mm512_permutex2var_epi32(v8, t5, v12);
            v8 = _mm512_permutex2var_epi32(v11, t6, v4);
            v12 = _mm512_permutex2var_epi32(v11, t7, v4);
            v4 = _mm512_permutex2var_epi32(v13, t6, v16);
            v11 = _mm512_permutex2var_epi32(v13, t7, v16);
            v13 = _mm512_permutex2var_epi32(v15, t6, v5);
            v16 = _mm512_permutex2var_epi32(v15, t7, v5);
            v5 = _mm512_permutex2var_epi32(v17, t6, v9);
            v15 = _mm512_permutex2var_epi32(v17, t7, v9);
            v9 = _mm512_permutex2var_epi32(v1, t6, v3);
            v17 = _mm512_permutex2var_epi32(v1, t7, v3);
            v1 = _mm512_permutex2var_epi32(v14, t6, v7);
            v3 = _mm512_permutex2var_epi32(v14, t7, v7);
            v7 = _mm512_permutex2var_epi32(v0, t6, v6);
            v14 = _mm512_permutex2var_epi32(v0, t7, v6);
            v0 = _mm512_permutex2var_epi32(v2, t6, v10);
            v6 = _mm512_permutex2var_epi32(v2, t7, v10);
            _mm512_store_epi32(dst + s0_d + 0, v8);
            _mm512_store_epi32(dst + s0_d + 4096, v13);
            _mm512_store_epi32(dst + s0_d + 8192, v9);
            _mm512_store_epi32(dst + s0_d + 12288, v7);
            _mm512_store_epi32(dst + s0_d + 16384, v4);
            _mm512_store_epi32(dst + s0_d + 20480, v5);
            _mm512_store_epi32(dst + s0_d + 24576, v1);
            _mm512_store_epi32(dst + s0_d + 28672, v0);
            _mm512_store_epi32(dst + s0_d + 32768, v12);
            _mm512_store_epi32(dst + s0_d + 36864, v16);
            _mm512_store_epi32(dst + s0_d + 40960, v17);
            _mm512_store_epi32(dst + s0_d + 45056, v14);
            _mm512_store_epi32(dst + s0_d + 49152, v11);
            _mm512_store_epi32(dst + s0_d + 53248, v15);
            _mm512_store_epi32(dst + s0_d + 57344, v3);
            _mm512_store_epi32(dst + s0_d + 61440, v6);
        }
    }
}
