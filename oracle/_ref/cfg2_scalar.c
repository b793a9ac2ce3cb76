/* generated vector permutation kernel
 * target: scalar  width: 512 bits  elem: 4 B  lanes: 16
 * shape (inner-first): (3136, 64, 32)  map (inner-first): (1, 0, 2)
 * shuffle steps: 4  block registers: 16  utilization: 1
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <string.h>
typedef uint32_t vp_elem_t;
static const int vp_tab0[16] = {0, 16, 2, 18, 4, 20, 6, 22, 8, 24, 10, 26, 12, 28, 14, 30};
static const int vp_tab1[16] = {1, 17, 3, 19, 5, 21, 7, 23, 9, 25, 11, 27, 13, 29, 15, 31};
static const int vp_tab2[16] = {0, 1, 16, 17, 4, 5, 20, 21, 8, 9, 24, 25, 12, 13, 28, 29};
static const int vp_tab3[16] = {2, 3, 18, 19, 6, 7, 22, 23, 10, 11, 26, 27, 14, 15, 30, 31};
static const int vp_tab4[16] = {0, 1, 2, 3, 16, 17, 18, 19, 8, 9, 10, 11, 24, 25, 26, 27};
static const int vp_tab5[16] = {4, 5, 6, 7, 20, 21, 22, 23, 12, 13, 14, 15, 28, 29, 30, 31};
static const int vp_tab6[16] = {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23};
static const int vp_tab7[16] = {8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31};
static void vp_adv_0(int64_t *i, int64_t *bs, int64_t *bd) {
    if (++i[0] < 4) { *bs += 50176; *bd += 16; return; }
    i[0] = 0; *bs -= 150528; *bd -= 48;
    if (++i[1] < 196) { *bs += 16; *bd += 1024; return; }
    i[1] = 0; *bs -= 3120; *bd -= 199680;
    if (++i[2] < 32) { *bs += 200704; *bd += 200704; return; }
    i[2] = 0; *bs -= 6221824; *bd -= 6221824;
}
void permute_22bdb72846c10e56(const void *src_v, void *dst_v) {
    const vp_elem_t *src = (const vp_elem_t *)src_v;
    vp_elem_t *dst = (vp_elem_t *)dst_v;
    { /* loop main: 25088 iterations, unroll 1 */
        int64_t vp_i[3] = {0, 0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        vp_elem_t v0[16];
        vp_elem_t v1[16];
        vp_elem_t v2[16];
        vp_elem_t v3[16];
        vp_elem_t v4[16];
        vp_elem_t v5[16];
        vp_elem_t v6[16];
        vp_elem_t v7[16];
        vp_elem_t v8[16];
        vp_elem_t v9[16];
        vp_elem_t v10[16];
        vp_elem_t v11[16];
        vp_elem_t v12[16];
        vp_elem_t v13[16];
        vp_elem_t v14[16];
        vp_elem_t v15[16];
        vp_elem_t v16[16];
        vp_elem_t v17[16];
        for (int64_t vp_it = 0; vp_it < 25088; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            memcpy(v0, src + s0_s + 0, sizeof(v0));
            memcpy(v1, src + s0_s + 3136, sizeof(v1));
            memcpy(v2, src + s0_s + 6272, sizeof(v2));
            memcpy(v3, src + s0_s + 9408, sizeof(v3));
            memcpy(v4, src + s0_s + 12544, sizeof(v4));
            memcpy(v5, src + s0_s + 15680, sizeof(v5));
            memcpy(v6, src + s0_s + 18816, sizeof(v6));
            memcpy(v7, src + s0_s + 21952, sizeof(v7));
            memcpy(v8, src + s0_s + 25088, sizeof(v8));
            memcpy(v9, src + s0_s + 28224, sizeof(v9));
            memcpy(v10, src + s0_s + 31360, sizeof(v10));
            memcpy(v11, src + s0_s + 34496, sizeof(v11));
            memcpy(v12, src + s0_s + 37632, sizeof(v12));
            memcpy(v13, src + s0_s + 40768, sizeof(v13));
            memcpy(v14, src + s0_s + 43904, sizeof(v14));
            memcpy(v15, src + s0_s + 47040, sizeof(v15));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v0[vp_tab0[k]] : v1[vp_tab0[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v0[vp_tab1[k]] : v1[vp_tab1[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v2[vp_tab0[k]] : v3[vp_tab0[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v2[vp_tab1[k]] : v3[vp_tab1[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v4[vp_tab0[k]] : v5[vp_tab0[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v4[vp_tab1[k]] : v5[vp_tab1[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v6[vp_tab0[k]] : v7[vp_tab0[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v6[vp_tab1[k]] : v7[vp_tab1[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v8[vp_tab0[k]] : v9[vp_tab0[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v8[vp_tab1[k]] : v9[vp_tab1[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v10[vp_tab0[k]] : v11[vp_tab0[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v10[vp_tab1[k]] : v11[vp_tab1[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v12[vp_tab0[k]] : v13[vp_tab0[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v12[vp_tab1[k]] : v13[vp_tab1[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v14[vp_tab0[k]] : v15[vp_tab0[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v14[vp_tab1[k]] : v15[vp_tab1[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v16[vp_tab2[k]] : v0[vp_tab2[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v16[vp_tab3[k]] : v0[vp_tab3[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v17[vp_tab2[k]] : v1[vp_tab2[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v17[vp_tab3[k]] : v1[vp_tab3[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v2[vp_tab2[k]] : v4[vp_tab2[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v2[vp_tab3[k]] : v4[vp_tab3[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v3[vp_tab2[k]] : v5[vp_tab2[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v3[vp_tab3[k]] : v5[vp_tab3[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v6[vp_tab2[k]] : v8[vp_tab2[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v6[vp_tab3[k]] : v8[vp_tab3[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v7[vp_tab2[k]] : v9[vp_tab2[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v7[vp_tab3[k]] : v9[vp_tab3[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v10[vp_tab2[k]] : v12[vp_tab2[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v10[vp_tab3[k]] : v12[vp_tab3[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab2[k] < 16 ? v11[vp_tab2[k]] : v13[vp_tab2[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab3[k] < 16 ? v11[vp_tab3[k]] : v13[vp_tab3[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v14[vp_tab4[k]] : v1[vp_tab4[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v14[vp_tab5[k]] : v1[vp_tab5[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v15[vp_tab4[k]] : v17[vp_tab4[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v15[vp_tab5[k]] : v17[vp_tab5[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v0[vp_tab4[k]] : v2[vp_tab4[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v0[vp_tab5[k]] : v2[vp_tab5[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v16[vp_tab4[k]] : v4[vp_tab4[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v16[vp_tab5[k]] : v4[vp_tab5[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v3[vp_tab4[k]] : v7[vp_tab4[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v3[vp_tab5[k]] : v7[vp_tab5[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v5[vp_tab4[k]] : v9[vp_tab4[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v5[vp_tab5[k]] : v9[vp_tab5[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v6[vp_tab4[k]] : v10[vp_tab4[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v6[vp_tab5[k]] : v10[vp_tab5[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v8[vp_tab4[k]] : v12[vp_tab4[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v8[vp_tab5[k]] : v12[vp_tab5[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v11[vp_tab6[k]] : v4[vp_tab6[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v11[vp_tab7[k]] : v4[vp_tab7[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v13[vp_tab6[k]] : v16[vp_tab6[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v13[vp_tab7[k]] : v16[vp_tab7[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v15[vp_tab6[k]] : v5[vp_tab6[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v15[vp_tab7[k]] : v5[vp_tab7[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v17[vp_tab6[k]] : v9[vp_tab6[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v17[vp_tab7[k]] : v9[vp_tab7[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v1[vp_tab6[k]] : v3[vp_tab6[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v1[vp_tab7[k]] : v3[vp_tab7[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v14[vp_tab6[k]] : v7[vp_tab6[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v14[vp_tab7[k]] : v7[vp_tab7[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v0[vp_tab6[k]] : v6[vp_tab6[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v0[vp_tab7[k]] : v6[vp_tab7[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v2[vp_tab6[k]] : v10[vp_tab6[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v2[vp_tab7[k]] : v10[vp_tab7[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 0, v8, sizeof(v8));
            memcpy(dst + s0_d + 64, v13, sizeof(v13));
            memcpy(dst + s0_d + 128, v9, sizeof(v9));
            memcpy(dst + s0_d + 192, v7, sizeof(v7));
            memcpy(dst + s0_d + 256, v4, sizeof(v4));
            memcpy(dst + s0_d + 320, v5, sizeof(v5));
            memcpy(dst + s0_d + 384, v1, sizeof(v1));
            memcpy(dst + s0_d + 448, v0, sizeof(v0));
            memcpy(dst + s0_d + 512, v12, sizeof(v12));
            memcpy(dst + s0_d + 576, v16, sizeof(v16));
            memcpy(dst + s0_d + 640, v17, sizeof(v17));
            memcpy(dst + s0_d + 704, v14, sizeof(v14));
            memcpy(dst + s0_d + 768, v11, sizeof(v11));
            memcpy(dst + s0_d + 832, v15, sizeof(v15));
            memcpy(dst + s0_d + 896, v3, sizeof(v3));
            memcpy(dst + s0_d + 960, v6, sizeof(v6));
        }
    }
}
