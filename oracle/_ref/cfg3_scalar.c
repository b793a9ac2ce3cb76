/* generated vector permutation kernel
 * target: scalar  width: 512 bits  elem: 4 B  lanes: 16
 * shape (inner-first): (27, 11, 15, 13, 9, 17)  map (inner-first): (2, 4, 1, 5, 3, 0)
 * shuffle steps: 4  block registers: 16  utilization: 405/512
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <string.h>
typedef uint32_t vp_elem_t;
static const int vp_tab0[16] = {0, 16, 2, 18, 4, 20, 6, 22, 8, 24, 10, 26, 12, 28, 14, 30};
static const int vp_tab1[16] = {1, 17, 3, 19, 5, 21, 7, 23, 9, 25, 11, 27, 13, 29, 15, 31};
static const int vp_tab2[16] = {0, 0, 2, 2, 4, 4, 6, 6, 8, 8, 10, 10, 12, 12, 14, 14};
static const int vp_tab3[16] = {1, 1, 3, 3, 5, 5, 7, 7, 9, 9, 11, 11, 13, 13, 15, 15};
static const int vp_tab4[16] = {0, 1, 16, 17, 4, 5, 20, 21, 8, 9, 24, 25, 12, 13, 28, 29};
static const int vp_tab5[16] = {2, 3, 18, 19, 6, 7, 22, 23, 10, 11, 26, 27, 14, 15, 30, 31};
static const int vp_tab6[16] = {0, 1, 2, 3, 16, 17, 18, 19, 8, 9, 10, 11, 24, 25, 26, 27};
static const int vp_tab7[16] = {4, 5, 6, 7, 20, 21, 22, 23, 12, 13, 14, 15, 28, 29, 30, 31};
static const int vp_tab8[16] = {0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23};
static const int vp_tab9[16] = {8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31};
static const int vp_tab10[16] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 31};
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
    const vp_elem_t *src = (const vp_elem_t *)src_v;
    vp_elem_t *dst = (vp_elem_t *)dst_v;
    { /* loop main: 21879 iterations, unroll 1 */
        int64_t vp_i[5] = {0, 0, 0, 0, 0};
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
        for (int64_t vp_it = 0; vp_it < 21879; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            memcpy(v0, src + s0_s + 0, sizeof(v0));
            memcpy(v1, src + s0_s + 297, sizeof(v1));
            memcpy(v2, src + s0_s + 594, sizeof(v2));
            memcpy(v3, src + s0_s + 891, sizeof(v3));
            memcpy(v4, src + s0_s + 1188, sizeof(v4));
            memcpy(v5, src + s0_s + 1485, sizeof(v5));
            memcpy(v6, src + s0_s + 1782, sizeof(v6));
            memcpy(v7, src + s0_s + 2079, sizeof(v7));
            memcpy(v8, src + s0_s + 2376, sizeof(v8));
            memcpy(v9, src + s0_s + 2673, sizeof(v9));
            memcpy(v10, src + s0_s + 2970, sizeof(v10));
            memcpy(v11, src + s0_s + 3267, sizeof(v11));
            memcpy(v12, src + s0_s + 3564, sizeof(v12));
            memcpy(v13, src + s0_s + 3861, sizeof(v13));
            memcpy(v14, src + s0_s + 4158, sizeof(v14));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v0[vp_tab0[k]] : v1[vp_tab0[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v0[vp_tab1[k]] : v1[vp_tab1[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
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
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = v14[vp_tab2[k]]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = v14[vp_tab3[k]]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v15[vp_tab4[k]] : v0[vp_tab4[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v15[vp_tab5[k]] : v0[vp_tab5[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v16[vp_tab4[k]] : v1[vp_tab4[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v16[vp_tab5[k]] : v1[vp_tab5[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v2[vp_tab4[k]] : v4[vp_tab4[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v2[vp_tab5[k]] : v4[vp_tab5[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v3[vp_tab4[k]] : v5[vp_tab4[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v3[vp_tab5[k]] : v5[vp_tab5[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v6[vp_tab4[k]] : v8[vp_tab4[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v6[vp_tab5[k]] : v8[vp_tab5[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v7[vp_tab4[k]] : v9[vp_tab4[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v7[vp_tab5[k]] : v9[vp_tab5[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v10[vp_tab4[k]] : v12[vp_tab4[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v10[vp_tab5[k]] : v12[vp_tab5[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v11[vp_tab4[k]] : v13[vp_tab4[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v11[vp_tab5[k]] : v13[vp_tab5[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v14[vp_tab6[k]] : v1[vp_tab6[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v14[vp_tab7[k]] : v1[vp_tab7[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v17[vp_tab6[k]] : v16[vp_tab6[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v17[vp_tab7[k]] : v16[vp_tab7[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v0[vp_tab6[k]] : v2[vp_tab6[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v0[vp_tab7[k]] : v2[vp_tab7[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v15[vp_tab6[k]] : v4[vp_tab6[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v15[vp_tab7[k]] : v4[vp_tab7[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v3[vp_tab6[k]] : v7[vp_tab6[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v3[vp_tab7[k]] : v7[vp_tab7[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v5[vp_tab6[k]] : v9[vp_tab6[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v5[vp_tab7[k]] : v9[vp_tab7[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v6[vp_tab6[k]] : v10[vp_tab6[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v6[vp_tab7[k]] : v10[vp_tab7[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v8[vp_tab6[k]] : v12[vp_tab6[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v8[vp_tab7[k]] : v12[vp_tab7[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v11[vp_tab8[k]] : v4[vp_tab8[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v11[vp_tab9[k]] : v4[vp_tab9[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v13[vp_tab8[k]] : v15[vp_tab8[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v13[vp_tab9[k]] : v15[vp_tab9[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v16[vp_tab8[k]] : v5[vp_tab8[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v16[vp_tab9[k]] : v5[vp_tab9[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v17[vp_tab8[k]] : v9[vp_tab8[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v17[vp_tab9[k]] : v9[vp_tab9[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v1[vp_tab8[k]] : v3[vp_tab8[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v1[vp_tab9[k]] : v3[vp_tab9[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v14[vp_tab8[k]] : v7[vp_tab8[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v14[vp_tab9[k]] : v7[vp_tab9[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v0[vp_tab8[k]] : v6[vp_tab8[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v0[vp_tab9[k]] : v6[vp_tab9[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v2[vp_tab8[k]] : v10[vp_tab8[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v2[vp_tab9[k]] : v10[vp_tab9[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(v2, dst + s0_d + 0, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v8[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 0, v10, sizeof(v10));
            memcpy(v2, dst + s0_d + 328185, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v13[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 328185, v8, sizeof(v8));
            memcpy(v2, dst + s0_d + 656370, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v9[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 656370, v8, sizeof(v8));
            memcpy(v2, dst + s0_d + 984555, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v7[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 984555, v8, sizeof(v8));
            memcpy(v2, dst + s0_d + 1312740, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v4[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1312740, v7, sizeof(v7));
            memcpy(v2, dst + s0_d + 1640925, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v5[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1640925, v4, sizeof(v4));
            memcpy(v2, dst + s0_d + 1969110, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v1[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1969110, v4, sizeof(v4));
            memcpy(v1, dst + s0_d + 2297295, sizeof(v1));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v0[vp_tab10[k]] : v1[vp_tab10[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2297295, v2, sizeof(v2));
            memcpy(v0, dst + s0_d + 2625480, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v12[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2625480, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 2953665, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v15[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2953665, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 3281850, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v17[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 3281850, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 3610035, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v14[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 3610035, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 3938220, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v11[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 3938220, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 4266405, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v16[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 4266405, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 4594590, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v3[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 4594590, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 4922775, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v6[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 4922775, v1, sizeof(v1));
        }
    }
    { /* loop tail[d0]: 21879 iterations, unroll 1 */
        int64_t vp_i[5] = {0, 0, 0, 0, 1};
        int64_t vp_bs = 16, vp_bd = 5250960;
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
        for (int64_t vp_it = 0; vp_it < 21879; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_1(vp_i, &vp_bs, &vp_bd);
            memcpy(v0, src + s0_s + 0, sizeof(v0));
            memcpy(v1, src + s0_s + 297, sizeof(v1));
            memcpy(v2, src + s0_s + 594, sizeof(v2));
            memcpy(v3, src + s0_s + 891, sizeof(v3));
            memcpy(v4, src + s0_s + 1188, sizeof(v4));
            memcpy(v5, src + s0_s + 1485, sizeof(v5));
            memcpy(v6, src + s0_s + 1782, sizeof(v6));
            memcpy(v7, src + s0_s + 2079, sizeof(v7));
            memcpy(v8, src + s0_s + 2376, sizeof(v8));
            memcpy(v9, src + s0_s + 2673, sizeof(v9));
            memcpy(v10, src + s0_s + 2970, sizeof(v10));
            memcpy(v11, src + s0_s + 3267, sizeof(v11));
            memcpy(v12, src + s0_s + 3564, sizeof(v12));
            memcpy(v13, src + s0_s + 3861, sizeof(v13));
            memcpy(v14, src + s0_s + 4158, sizeof(v14));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab0[k] < 16 ? v0[vp_tab0[k]] : v1[vp_tab0[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab1[k] < 16 ? v0[vp_tab1[k]] : v1[vp_tab1[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
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
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = v14[vp_tab2[k]]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = v14[vp_tab3[k]]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v15[vp_tab4[k]] : v0[vp_tab4[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v15[vp_tab5[k]] : v0[vp_tab5[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v16[vp_tab4[k]] : v1[vp_tab4[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v16[vp_tab5[k]] : v1[vp_tab5[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v2[vp_tab4[k]] : v4[vp_tab4[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v2[vp_tab5[k]] : v4[vp_tab5[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v3[vp_tab4[k]] : v5[vp_tab4[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v3[vp_tab5[k]] : v5[vp_tab5[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v6[vp_tab4[k]] : v8[vp_tab4[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v6[vp_tab5[k]] : v8[vp_tab5[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v7[vp_tab4[k]] : v9[vp_tab4[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v7[vp_tab5[k]] : v9[vp_tab5[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v10[vp_tab4[k]] : v12[vp_tab4[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v10[vp_tab5[k]] : v12[vp_tab5[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab4[k] < 16 ? v11[vp_tab4[k]] : v13[vp_tab4[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab5[k] < 16 ? v11[vp_tab5[k]] : v13[vp_tab5[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v14[vp_tab6[k]] : v1[vp_tab6[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v14[vp_tab7[k]] : v1[vp_tab7[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v17[vp_tab6[k]] : v16[vp_tab6[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v17[vp_tab7[k]] : v16[vp_tab7[k] - 16]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v0[vp_tab6[k]] : v2[vp_tab6[k] - 16]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v0[vp_tab7[k]] : v2[vp_tab7[k] - 16]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v15[vp_tab6[k]] : v4[vp_tab6[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v15[vp_tab7[k]] : v4[vp_tab7[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v3[vp_tab6[k]] : v7[vp_tab6[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v3[vp_tab7[k]] : v7[vp_tab7[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v5[vp_tab6[k]] : v9[vp_tab6[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v5[vp_tab7[k]] : v9[vp_tab7[k] - 16]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v6[vp_tab6[k]] : v10[vp_tab6[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v6[vp_tab7[k]] : v10[vp_tab7[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab6[k] < 16 ? v8[vp_tab6[k]] : v12[vp_tab6[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab7[k] < 16 ? v8[vp_tab7[k]] : v12[vp_tab7[k] - 16]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v11[vp_tab8[k]] : v4[vp_tab8[k] - 16]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v11[vp_tab9[k]] : v4[vp_tab9[k] - 16]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v13[vp_tab8[k]] : v15[vp_tab8[k] - 16]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v16[vp_tab8[k]] : v5[vp_tab8[k] - 16]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v16[vp_tab9[k]] : v5[vp_tab9[k] - 16]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v17[vp_tab8[k]] : v9[vp_tab8[k] - 16]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v1[vp_tab8[k]] : v3[vp_tab8[k] - 16]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab9[k] < 16 ? v1[vp_tab9[k]] : v3[vp_tab9[k] - 16]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v14[vp_tab8[k]] : v7[vp_tab8[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v0[vp_tab8[k]] : v6[vp_tab8[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab8[k] < 16 ? v2[vp_tab8[k]] : v10[vp_tab8[k] - 16]; memcpy(v0, vp_t, sizeof(vp_t)); }
            memcpy(v2, dst + s0_d + 0, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v8[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 0, v6, sizeof(v6));
            memcpy(v2, dst + s0_d + 328185, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v11[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 328185, v6, sizeof(v6));
            memcpy(v2, dst + s0_d + 656370, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v9[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 656370, v6, sizeof(v6));
            memcpy(v2, dst + s0_d + 984555, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v3[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v6, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 984555, v6, sizeof(v6));
            memcpy(v2, dst + s0_d + 1312740, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v4[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1312740, v3, sizeof(v3));
            memcpy(v2, dst + s0_d + 1640925, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v5[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1640925, v3, sizeof(v3));
            memcpy(v2, dst + s0_d + 1969110, sizeof(v2));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v1[vp_tab10[k]] : v2[vp_tab10[k] - 16]; memcpy(v3, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 1969110, v3, sizeof(v3));
            memcpy(v1, dst + s0_d + 2297295, sizeof(v1));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v0[vp_tab10[k]] : v1[vp_tab10[k] - 16]; memcpy(v2, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2297295, v2, sizeof(v2));
            memcpy(v0, dst + s0_d + 2625480, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v12[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2625480, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 2953665, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v13[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 2953665, v1, sizeof(v1));
            memcpy(v0, dst + s0_d + 3281850, sizeof(v0));
            { vp_elem_t vp_t[16]; int k; for (k = 0; k < 16; ++k) vp_t[k] = vp_tab10[k] < 16 ? v15[vp_tab10[k]] : v0[vp_tab10[k] - 16]; memcpy(v1, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 3281850, v1, sizeof(v1));
        }
    }
}
