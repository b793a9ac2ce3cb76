/* generated vector permutation kernel
 * target: x86-avx  width: 512 bits  elem: 4 B  lanes: 16
 * shape (inner-first): (27, 11, 15, 13, 9, 17)  map (inner-first): (2, 4, 1, 5, 3, 0)
 * shuffle steps: 4  block registers: 16  utilization: 405/512
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <immintrin.h>
static const uint32_t vp_tab0[16] = {0, 16, 2, 18, 4, 20, 6, 22, 8, 24, 10, 26, 12, 28, 14, 30};
static const uint32_t vp_tab1[16] = {1, 17, 3, 19, 5, 21, 7, 23, 9, 25, 11, 27, 13, 29, 15, 31};
static const uint32_t vp_tab2[16] = {0, 0, 2, 2, 4, 4, 6, 6, 8, 8, 10, 10, 12, 12, 14, 14};
static const uint32_t vp_tab3[16] = {1, 1, 3, 3, 5, 5, 7, 7, 9, 9, 11, 11, 13, 13, 15, 15};
static const uint32_t vp_tab4[16] = {0, 1, 16, 17, 4, 5, 20, 21, 8, 9, 24, 25, 12, 13, 28, 29};
static const uint32_t vp_tab5[16] = {2, 3, 18, 19, 6, 7, 22, 23, 10, 11, 26, 27, 14, 15, 30, 31};
static const uint32_t vp_tab6[16] = {0, 1, 2, 3, 16, 17, 18, 19, 8, 9, 10, 11, 24, 25, 26, 27};
static const uint32_t vp_tab7[16] = {4, 5, 6, 7, 20, 21, 22, 23, 12, 13, 14, 15, 28, 29, 30, 31};
static const uint32_t vp_tab8[16] = {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23};
static const uint32_t vp_tab9[16] = {8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31};
static const uint32_t vp_tab10[16] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 31};
static void vp_adv_0(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 9) { *bs += 57915; *bd += 15; return; }
    i[0] = 0; *bs -= 463320; *bd -= 120;
    if (++i[1] < 11) { *bs += 27; *bd += 135; return; }
    i[1] = 0; *bs -= 270; *bd -= 1350;
    if (++i[2] < 17) { *bs += 521235; *bd += 1485; return; }
    i[2] = 0; *bs -= 8339760; *bd -= 23760;
    if (++i[3] < 13) { *bs += 4455; *bd += 25245; return; }
    i[3] = 0; *bs -= 53460; *bd -= 302940;
    if (++i[4] < 1) { *bs += 16; *bd += 5250960; return; }
    i[4] = 0; *bs -= 0; *bd -= 0;
}
static void vp_adv_1(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 9) { *bs += 57915; *bd += 15; return; }
    i[0] = 0; *bs -= 463320; *bd -= 120;
    if (++i[1] < 11) { *bs += 27; *bd += 135; return; }
    i[1] = 0; *bs -= 270; *bd -= 1350;
    if (++i[2] < 17) { *bs += 521235; *bd += 1485; return; }
    i[2] = 0; *bs -= 8339760; *bd -= 23760;
    if (++i[3] < 13) { *bs += 4455; *bd += 25245; return; }
    i[3] = 0; *bs -= 53460; *bd -= 302940;
    if (++i[4] < 2) { *bs += 16; *bd += 5250960; return; }
    i[4] = 1; *bs -= 0; *bd -= 0;
}
void permute_30fb771ec8238d2a(const void *src_v, void *dst_v) {
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
    const __m512i t8 = _mm512_loadu_epi32(vp_tab8);
    const __m512i t9 = _mm512_loadu_epi32(vp_tab9);
    const __m512i t10 = _mm512_loadu_epi32(vp_tab10);
    { /* loop main: 21879 iterations, unroll 1 */
        int64_t vp_i[5] = {0, 0, 0, 0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        __m512i v0, v1, v2, v3, v4, v5, v6, v7, v8, v9, v10, v11, v12, v13, v14, v15, v16, v17;
        for (int64_t vp_it = 0; vp_it < 21879; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            v0 = _mm512_loadu_epi32(src + s0_s + 0);
            v1 = _mm512_loadu_epi32(src + s0_s + 297);
            v2 = _mm512_loadu_epi32(src + s0_s + 594);
            v3 = _mm512_loadu_epi32(src + s0_s + 891);
            v4 = _mm512_loadu_epi32(src + s0_s + 1188);
            v5 = _mm512_loadu_epi32(src + s0_s + 1485);
            v6 = _mm512_loadu_epi32(src + s0_s + 1782);
            v7 = _mm512_loadu_epi32(src + s0_s + 2079);
            v8 = _mm512_loadu_epi32(src + s0_s + 2376);
            v9 = _mm512_loadu_epi32(src + s0_s + 2673);
            v10 = _mm512_loadu_epi32(src + s0_s + 2970);
            v11 = _mm512_loadu_epi32(src + s0_s + 3267);
            v12 = _mm512_loadu_epi32(src + s0_s + 3564);
            v13 = _mm512_loadu_epi32(src + s0_s + 3861);
            v14 = _mm512_loadu_epi32(src + s0_s + 4158);
            v15 = _mm512_permutex2var_epi32(v0, t0, v1);
            v16 = _mm512_permutex2var_epi32(v0, t1, v1);
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
            v12 = _mm512_permutexvar_epi32(t2, v14);
            v13 = _mm512_permutexvar_epi32(t3, v14);
            v14 = _mm512_permutex2var_epi32(v15, t4, v0);
            v17 = _mm512_permutex2var_epi32(v15, t5, v0);
            v0 = _mm512_permutex2var_epi32(v16, t4, v1);
            v15 = _mm512_permutex2var_epi32(v16, t5, v1);
            v1 = _mm512_permutex2var_epi32(v2, t4, v4);
            v16 = _mm512_permutex2var_epi32(v2, t5, v4);
            v2 = _mm512_permutex2var_epi32(v3, t4, v5);
            v4 = _mm512_permutex2var_epi32(v3, t5, v5);
            v3 = _mm512_permutex2var_epi32(v6, t4, v8);
            v5 = _mm512_permutex2var_epi32(v6, t5, v8);
            v6 = _mm512_permutex2var_epi32(v7, t4, v9);
            v8 = _mm512_permutex2var_epi32(v7, t5, v9);
            v7 = _mm512_permutex2var_epi32(v10, t4, v12);
            v9 = _mm512_permutex2var_epi32(v10, t5, v12);
            v10 = _mm512_permutex2var_epi32(v11, t4, v13);
            v12 = _mm512_permutex2var_epi32(v11, t5, v13);
            v11 = _mm512_permutex2var_epi32(v14, t6, v1);
            v13 = _mm512_permutex2var_epi32(v14, t7, v1);
            v1 = _mm512_permutex2var_epi32(v17, t6, v16);
            v14 = _mm512_permutex2var_epi32(v17, t7, v16);
            v16 = _mm512_permutex2var_epi32(v0, t6, v2);
            v17 = _mm512_permutex2var_epi32(v0, t7, v2);
            v0 = _mm512_permutex2var_epi32(v15, t6, v4);
            v2 = _mm512_permutex2var_epi32(v15, t7, v4);
            v4 = _mm512_permutex2var_epi32(v3, t6, v7);
            v15 = _mm512_permutex2var_epi32(v3, t7, v7);
            v3 = _mm512_permutex2var_epi32(v5, t6, v9);
            v7 = _mm512_permutex2var_epi32(v5, t7, v9);
            v5 = _mm512_permutex2var_epi32(v6, t6, v10);
            v9 = _mm512_permutex2var_epi32(v6, t7, v10);
            v6 = _mm512_permutex2var_epi32(v8, t6, v12);
            v10 = _mm512_permutex2var_epi32(v8, t7, v12);
            v8 = _mm512_permutex2var_epi32(v11, t8, v4);
            v12 = _mm512_permutex2var_epi32(v11, t9, v4);
            v4 = _mm512_permutex2var_epi32(v13, t8, v15);
            v11 = _mm512_permutex2var_epi32(v13, t9, v15);
            v13 = _mm512_permutex2var_epi32(v16, t8, v5);
            v15 = _mm512_permutex2var_epi32(v16, t9, v5);
            v5 = _mm512_permutex2var_epi32(v17, t8, v9);
            v16 = _mm512_permutex2var_epi32(v17, t9, v9);
            v9 = _mm512_permutex2var_epi32(v1, t8, v3);
            v17 = _mm512_permutex2var_epi32(v1, t9, v3);
            v1 = _mm512_permutex2var_epi32(v14, t8, v7);
            v3 = _mm512_permutex2var_epi32(v14, t9, v7);
            v7 = _mm512_permutex2var_epi32(v0, t8, v6);
            v14 = _mm512_permutex2var_epi32(v0, t9, v6);
            v0 = _mm512_permutex2var_epi32(v2, t8, v10);
            v6 = _mm512_permutex2var_epi32(v2, t9, v10);
            v2 = _mm512_loadu_epi32(dst + s0_d + 0);
            v10 = _mm512_permutex2var_epi32(v8, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 0, v10);
            v2 = _mm512_loadu_epi32(dst + s0_d + 328185);
            v8 = _mm512_permutex2var_epi32(v13, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 328185, v8);
            v2 = _mm512_loadu_epi32(dst + s0_d + 656370);
            v8 = _mm512_permutex2var_epi32(v9, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 656370, v8);
            v2 = _mm512_loadu_epi32(dst + s0_d + 984555);
            v8 = _mm512_permutex2var_epi32(v7, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 984555, v8);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1312740);
            v7 = _mm512_permutex2var_epi32(v4, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1312740, v7);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1640925);
            v4 = _mm512_permutex2var_epi32(v5, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1640925, v4);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1969110);
            v4 = _mm512_permutex2var_epi32(v1, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1969110, v4);
            v1 = _mm512_loadu_epi32(dst + s0_d + 2297295);
            v2 = _mm512_permutex2var_epi32(v0, t10, v1);
            _mm512_storeu_epi32(dst + s0_d + 2297295, v2);
            v0 = _mm512_loadu_epi32(dst + s0_d + 2625480);
            v1 = _mm512_permutex2var_epi32(v12, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 2625480, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 2953665);
            v1 = _mm512_permutex2var_epi32(v15, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 2953665, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 3281850);
            v1 = _mm512_permutex2var_epi32(v17, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 3281850, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 3610035);
            v1 = _mm512_permutex2var_epi32(v14, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 3610035, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 3938220);
            v1 = _mm512_permutex2var_epi32(v11, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 3938220, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 4266405);
            v1 = _mm512_permutex2var_epi32(v16, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 4266405, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 4594590);
            v1 = _mm512_permutex2var_epi32(v3, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 4594590, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 4922775);
            v1 = _mm512_permutex2var_epi32(v6, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 4922775, v1);
        }
    }
    { /* loop tail[d0]: 21879 iterations, unroll 1 */
        int64_t vp_i[5] = {0, 0, 0, 0, 1};
        int64_t vp_bs = 16, vp_bd = 5250960;
        int64_t s0_s = 0, s0_d = 0;
        __m512i v0, v1, v2, v3, v4, v5, v6, v7, v8, v9, v10, v11, v12, v13, v14, v15, v16, v17;
        for (int64_t vp_it = 0; vp_it < 21879; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_1(vp_i, &vp_bs, &vp_bd);
            v0 = _mm512_loadu_epi32(src + s0_s + 0);
            v1 = _mm512_loadu_epi32(src + s0_s + 297);
            v2 = _mm512_loadu_epi32(src + s0_s + 594);
            v3 = _mm512_loadu_epi32(src + s0_s + 891);
            v4 = _mm512_loadu_epi32(src + s0_s + 1188);
            v5 = _mm512_loadu_epi32(src + s0_s + 1485);
            v6 = _mm512_loadu_epi32(src + s0_s + 1782);
            v7 = _mm512_loadu_epi32(src + s0_s + 2079);
            v8 = _mm512_loadu_epi32(src + s0_s + 2376);
            v9 = _mm512_loadu_epi32(src + s0_s + 2673);
            v10 = _mm512_loadu_epi32(src + s0_s + 2970);
            v11 = _mm512_loadu_epi32(src + s0_s + 3267);
            v12 = _mm512_loadu_epi32(src + s0_s + 3564);
            v13 = _mm512_loadu_epi32(src + s0_s + 3861);
            v14 = _mm512_loadu_epi32(src + s0_s + 4158);
            v15 = _mm512_permutex2var_epi32(v0, t0, v1);
            v16 = _mm512_permutex2var_epi32(v0, t1, v1);
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
            v12 = _mm512_permutexvar_epi32(t2, v14);
            v13 = _mm512_permutexvar_epi32(t3, v14);
            v14 = _mm512_permutex2var_epi32(v15, t4, v0);
            v17 = _mm512_permutex2var_epi32(v15, t5, v0);
            v0 = _mm512_permutex2var_epi32(v16, t4, v1);
            v15 = _mm512_permutex2var_epi32(v16, t5, v1);
            v1 = _mm512_permutex2var_epi32(v2, t4, v4);
            v16 = _mm512_permutex2var_epi32(v2, t5, v4);
            v2 = _mm512_permutex2var_epi32(v3, t4, v5);
            v4 = _mm512_permutex2var_epi32(v3, t5, v5);
            v3 = _mm512_permutex2var_epi32(v6, t4, v8);
            v5 = _mm512_permutex2var_epi32(v6, t5, v8);
            v6 = _mm512_permutex2var_epi32(v7, t4, v9);
            v8 = _mm512_permutex2var_epi32(v7, t5, v9);
            v7 = _mm512_permutex2var_epi32(v10, t4, v12);
            v9 = _mm512_permutex2var_epi32(v10, t5, v12);
            v10 = _mm512_permutex2var_epi32(v11, t4, v13);
            v12 = _mm512_permutex2var_epi32(v11, t5, v13);
            v11 = _mm512_permutex2var_epi32(v14, t6, v1);
            v13 = _mm512_permutex2var_epi32(v14, t7, v1);
            v1 = _mm512_permutex2var_epi32(v17, t6, v16);
            v14 = _mm512_permutex2var_epi32(v17, t7, v16);
            v16 = _mm512_permutex2var_epi32(v0, t6, v2);
            v17 = _mm512_permutex2var_epi32(v0, t7, v2);
            v0 = _mm512_permutex2var_epi32(v15, t6, v4);
            v2 = _mm512_permutex2var_epi32(v15, t7, v4);
            v4 = _mm512_permutex2var_epi32(v3, t6, v7);
            v15 = _mm512_permutex2var_epi32(v3, t7, v7);
            v3 = _mm512_permutex2var_epi32(v5, t6, v9);
            v7 = _mm512_permutex2var_epi32(v5, t7, v9);
            v5 = _mm512_permutex2var_epi32(v6, t6, v10);
            v9 = _mm512_permutex2var_epi32(v6, t7, v10);
            v6 = _mm512_permutex2var_epi32(v8, t6, v12);
            v10 = _mm512_permutex2var_epi32(v8, t7, v12);
            v8 = _mm512_permutex2var_epi32(v11, t8, v4);
            v12 = _mm512_permutex2var_epi32(v11, t9, v4);
            v4 = _mm512_permutex2var_epi32(v13, t8, v15);
            v11 = _mm512_permutex2var_epi32(v16, t8, v5);
            v13 = _mm512_permutex2var_epi32(v16, t9, v5);
            v5 = _mm512_permutex2var_epi32(v17, t8, v9);
            v9 = _mm512_permutex2var_epi32(v1, t8, v3);
            v15 = _mm512_permutex2var_epi32(v1, t9, v3);
            v1 = _mm512_permutex2var_epi32(v14, t8, v7);
            v3 = _mm512_permutex2var_epi32(v0, t8, v6);
            v0 = _mm512_permutex2var_epi32(v2, t8, v10);
            v2 = _mm512_loadu_epi32(dst + s0_d + 0);
            v6 = _mm512_permutex2var_epi32(v8, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 0, v6);
            v2 = _mm512_loadu_epi32(dst + s0_d + 328185);
            v6 = _mm512_permutex2var_epi32(v11, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 328185, v6);
            v2 = _mm512_loadu_epi32(dst + s0_d + 656370);
            v6 = _mm512_permutex2var_epi32(v9, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 656370, v6);
            v2 = _mm512_loadu_epi32(dst + s0_d + 984555);
            v6 = _mm512_permutex2var_epi32(v3, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 984555, v6);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1312740);
            v3 = _mm512_permutex2var_epi32(v4, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1312740, v3);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1640925);
            v3 = _mm512_permutex2var_epi32(v5, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1640925, v3);
            v2 = _mm512_loadu_epi32(dst + s0_d + 1969110);
            v3 = _mm512_permutex2var_epi32(v1, t10, v2);
            _mm512_storeu_epi32(dst + s0_d + 1969110, v3);
            v1 = _mm512_loadu_epi32(dst + s0_d + 2297295);
            v2 = _mm512_permutex2var_epi32(v0, t10, v1);
            _mm512_storeu_epi32(dst + s0_d + 2297295, v2);
            v0 = _mm512_loadu_epi32(dst + s0_d + 2625480);
            v1 = _mm512_permutex2var_epi32(v12, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 2625480, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 2953665);
            v1 = _mm512_permutex2var_epi32(v13, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 2953665, v1);
            v0 = _mm512_loadu_epi32(dst + s0_d + 3281850);
            v1 = _mm512_permutex2var_epi32(v15, t10, v0);
            _mm512_storeu_epi32(dst + s0_d + 3281850, v1);
        }
    }
}
