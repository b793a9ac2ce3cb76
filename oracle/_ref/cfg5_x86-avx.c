/* generated vector permutation kernel
 * target: x86-avx  width: 512 bits  elem: 8 B  lanes: 8
 * shape (inner-first): (2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 4, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2)  map (inner-first): (12, 25, 3, 2, 17, 5, 13, 10, 21, 19, 14, 9, 15, 7, 26, 18, 6, 23, 4, 11, 20, 1, 24, 0, 16, 22, 8)
 * shuffle steps: 3  block registers: 8  utilization: 1
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <immintrin.h>
static const uint32_t vp_tab0[16] = {0, 1, 16, 17, 4, 5, 20, 21, 8, 9, 24, 25, 12, 13, 28, 29};
static const uint32_t vp_tab1[16] = {2, 3, 18, 19, 6, 7, 22, 23, 10, 11, 26, 27, 14, 15, 30, 31};
static const uint32_t vp_tab2[16] = {0, 1, 2, 3, 16, 17, 18, 19, 8, 9, 10, 11, 24, 25, 26, 27};
static const uint32_t vp_tab3[16] = {4, 5, 6, 7, 20, 21, 22, 23, 12, 13, 14, 15, 28, 29, 30, 31};
static const uint32_t vp_tab4[16] = {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23};
static const uint32_t vp_tab5[16] = {8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31};
static void vp_adv_0(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 2) { *bs += 262144; *bd += 16; return; }
    i[0] = 0; *bs -= 262144; *bd -= 16;
    if (++i[1] < 2) { *bs += 32; *bd += 32; return; }
    i[1] = 0; *bs -= 32; *bd -= 32;
    if (++i[2] < 2) { *bs += 8192; *bd += 64; return; }
    i[2] = 0; *bs -= 8192; *bd -= 64;
    if (++i[3] < 2) { *bs += 1024; *bd += 128; return; }
    i[3] = 0; *bs -= 1024; *bd -= 128;
    if (++i[4] < 2) { *bs += 4194304; *bd += 256; return; }
    i[4] = 0; *bs -= 4194304; *bd -= 256;
    if (++i[5] < 2) { *bs += 1048576; *bd += 512; return; }
    i[5] = 0; *bs -= 1048576; *bd -= 512;
    if (++i[6] < 2) { *bs += 16384; *bd += 1024; return; }
    i[6] = 0; *bs -= 16384; *bd -= 1024;
    if (++i[7] < 2) { *bs += 512; *bd += 2048; return; }
    i[7] = 0; *bs -= 512; *bd -= 2048;
    if (++i[8] < 2) { *bs += 32768; *bd += 4096; return; }
    i[8] = 0; *bs -= 32768; *bd -= 4096;
    if (++i[9] < 2) { *bs += 128; *bd += 8192; return; }
    i[9] = 0; *bs -= 128; *bd -= 8192;
    if (++i[10] < 2) { *bs += 134217728; *bd += 16384; return; }
    i[10] = 0; *bs -= 134217728; *bd -= 16384;
    if (++i[11] < 2) { *bs += 524288; *bd += 32768; return; }
    i[11] = 0; *bs -= 524288; *bd -= 32768;
    if (++i[12] < 2) { *bs += 64; *bd += 65536; return; }
    i[12] = 0; *bs -= 64; *bd -= 65536;
    if (++i[13] < 2) { *bs += 16777216; *bd += 131072; return; }
    i[13] = 0; *bs -= 16777216; *bd -= 131072;
    if (++i[14] < 2) { *bs += 16; *bd += 262144; return; }
    i[14] = 0; *bs -= 16; *bd -= 262144;
    if (++i[15] < 2) { *bs += 2048; *bd += 524288; return; }
    i[15] = 0; *bs -= 2048; *bd -= 524288;
    if (++i[16] < 2) { *bs += 2097152; *bd += 1048576; return; }
    i[16] = 0; *bs -= 2097152; *bd -= 1048576;
    if (++i[17] < 2) { *bs += 33554432; *bd += 4194304; return; }
    i[17] = 0; *bs -= 33554432; *bd -= 4194304;
    if (++i[18] < 4) { *bs += 65536; *bd += 16777216; return; }
    i[18] = 0; *bs -= 196608; *bd -= 50331648;
    if (++i[19] < 2) { *bs += 8388608; *bd += 67108864; return; }
    i[19] = 0; *bs -= 8388608; *bd -= 67108864;
    if (++i[20] < 2) { *bs += 256; *bd += 134217728; return; }
    i[20] = 0; *bs -= 256; *bd -= 134217728;
}
void permute_d05b2e98286551f4(const void *src_v, void *dst_v) {
    const uint32_t *src = (const uint32_t *)src_v;
    uint32_t *dst = (uint32_t *)dst_v;
    const __m512i t0 = _mm512_loadu_epi32(vp_tab0);
    const __m512i t1 = _mm512_loadu_epi32(vp_tab1);
    const __m512i t2 = _mm512_loadu_epi32(vp_tab2);
    const __m512i t3 = _mm512_loadu_epi32(vp_tab3);
    const __m512i t4 = _mm512_loadu_epi32(vp_tab4);
    const __m512i t5 = _mm512_loadu_epi32(vp_tab5);
    { /* loop main: 2097152 iterations, unroll 2 */
        int64_t vp_i[21] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        int64_t s1_s = 0, s1_d = 0;
        __m512i v0, v1, v2, v3, v4, v5, v6, v7, v8, v9, v10, v11, v12, v13, v14, v15, v16, v17;
        for (int64_t vp_it = 0; vp_it < 2097152; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s1_s = vp_bs; s1_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            v0 = _mm512_load_epi32(src + (s0_s + 0) * 2);
            v1 = _mm512_load_epi32(src + (s0_s + 4096) * 2);
            v2 = _mm512_load_epi32(src + (s0_s + 67108864) * 2);
            v3 = _mm512_load_epi32(src + (s0_s + 67112960) * 2);
            v4 = _mm512_load_epi32(src + (s0_s + 8) * 2);
            v5 = _mm512_load_epi32(src + (s0_s + 4104) * 2);
            v6 = _mm512_load_epi32(src + (s0_s + 67108872) * 2);
            v7 = _mm512_load_epi32(src + (s0_s + 67112968) * 2);
            v8 = _mm512_load_epi32(src + (s1_s + 0) * 2);
            v9 = _mm512_load_epi32(src + (s1_s + 4096) * 2);
            v10 = _mm512_load_epi32(src + (s1_s + 67108864) * 2);
            v11 = _mm512_load_epi32(src + (s1_s + 67112960) * 2);
            v12 = _mm512_load_epi32(src + (s1_s + 8) * 2);
            v13 = _mm512_load_epi32(src + (s1_s + 4104) * 2);
            v14 = _mm512_load_epi32(src + (s1_s + 67108872) * 2);
            v15 = _mm512_load_epi32(src + (s1_s + 67112968) * 2);
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
            v3 = _mm512_permutex2var_epi32(v14, t4, v1);
            v5 = _mm512_permutex2var_epi32(v14, t5, v1);
            v1 = _mm512_permutex2var_epi32(v15, t4, v17);
            v14 = _mm512_permutex2var_epi32(v15, t5, v17);
            v15 = _mm512_permutex2var_epi32(v0, t4, v2);
            v17 = _mm512_permutex2var_epi32(v0, t5, v2);
            v0 = _mm512_permutex2var_epi32(v16, t4, v4);
            v2 = _mm512_permutex2var_epi32(v16, t5, v4);
            v4 = _mm512_permutex2var_epi32(v6, t2, v8);
            v16 = _mm512_permutex2var_epi32(v6, t3, v8);
            v6 = _mm512_permutex2var_epi32(v7, t2, v9);
            v8 = _mm512_permutex2var_epi32(v7, t3, v9);
            v7 = _mm512_permutex2var_epi32(v10, t2, v12);
            v9 = _mm512_permutex2var_epi32(v10, t3, v12);
            v10 = _mm512_permutex2var_epi32(v11, t2, v13);
            v12 = _mm512_permutex2var_epi32(v11, t3, v13);
            v11 = _mm512_permutex2var_epi32(v4, t4, v7);
            v13 = _mm512_permutex2var_epi32(v4, t5, v7);
            v4 = _mm512_permutex2var_epi32(v16, t4, v9);
            v7 = _mm512_permutex2var_epi32(v16, t5, v9);
            v9 = _mm512_permutex2var_epi32(v6, t4, v10);
            v16 = _mm512_permutex2var_epi32(v6, t5, v10);
            v6 = _mm512_permutex2var_epi32(v8, t4, v12);
            v10 = _mm512_permutex2var_epi32(v8, t5, v12);
            _mm512_store_epi32(dst + (s0_d + 0) * 2, v3);
            _mm512_store_epi32(dst + (s0_d + 8) * 2, v5);
            _mm512_store_epi32(dst + (s0_d + 2097152) * 2, v1);
            _mm512_store_epi32(dst + (s0_d + 2097160) * 2, v14);
            _mm512_store_epi32(dst + (s0_d + 8388608) * 2, v15);
            _mm512_store_epi32(dst + (s0_d + 8388616) * 2, v17);
            _mm512_store_epi32(dst + (s0_d + 10485760) * 2, v0);
            _mm512_store_epi32(dst + (s0_d + 10485768) * 2, v2);
            _mm512_store_epi32(dst + (s1_d + 0) * 2, v11);
            _mm512_store_epi32(dst + (s1_d + 8) * 2, v13);
            _mm512_store_epi32(dst + (s1_d + 2097152) * 2, v4);
            _mm512_store_epi32(dst + (s1_d + 2097160) * 2, v7);
            _mm512_store_epi32(dst + (s1_d + 8388608) * 2, v9);
            _mm512_store_epi32(dst + (s1_d + 8388616) * 2, v16);
            _mm512_store_epi32(dst + (s1_d + 10485760) * 2, v6);
            _mm512_store_epi32(dst + (s1_d + 10485768) * 2, v10);
        }
    }
}
