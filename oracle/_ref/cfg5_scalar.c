/* generated vector permutation kernel
 * target: scalar  width: 512 bits  elem: 8 B  lanes: 8
 * shape (inner-first): (2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2, 4, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2)  map (inner-first): (12, 25, 3, 2, 17, 5, 13, 10, 21, 19, 14, 9, 15, 7, 26, 18, 6, 23, 4, 11, 20, 1, 24, 0, 16, 22, 8)
 * shuffle steps: 3  block registers: 8  utilization: 1
 * buffers need one vector width of writable slack past the data;
 * aligned accesses, when present, assume vector-aligned buffer bases
 */
#include <stdint.h>
#include <string.h>
typedef uint64_t vp_elem_t;
static const int vp_tab0[8] = {0, 8, 2, 10, 4, 12, 6, 14};
static const int vp_tab1[8] = {1, 9, 3, 11, 5, 13, 7, 15};
static const int vp_tab2[8] = {0, 1, 8, 9, 4, 5, 12, 13};
static const int vp_tab3[8] = {2, 3, 10, 11, 6, 7, 14, 15};
static const int vp_tab4[8] = {0, 1, 2, 3, 8, 9, 10, 11};
static const int vp_tab5[8] = {4, 5, 6, 7, 12, 13, 14, 15};
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
    const vp_elem_t *src = (const vp_elem_t *)src_v;
    vp_elem_t *dst = (vp_elem_t *)dst_v;
    { /* loop main: 2097152 iterations, unroll 2 */
        int64_t vp_i[21] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        int64_t vp_bs = 0, vp_bd = 0;
        int64_t s0_s = 0, s0_d = 0;
        int64_t s1_s = 0, s1_d = 0;
        vp_elem_t v0[8];
        vp_elem_t v1[8];
        vp_elem_t v2[8];
        vp_elem_t v3[8];
        vp_elem_t v4[8];
        vp_elem_t v5[8];
        vp_elem_t v6[8];
        vp_elem_t v7[8];
        vp_elem_t v8[8];
        vp_elem_t v9[8];
        vp_elem_t v10[8];
        vp_elem_t v11[8];
        vp_elem_t v12[8];
        vp_elem_t v13[8];
        vp_elem_t v14[8];
        vp_elem_t v15[8];
        vp_elem_t v16[8];
        vp_elem_t v17[8];
        for (int64_t vp_it = 0; vp_it < 2097152; ++vp_it) {
            s0_s = vp_bs; s0_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            s1_s = vp_bs; s1_d = vp_bd; vp_adv_0(vp_i, &vp_bs, &vp_bd);
            memcpy(v0, src + s0_s + 0, sizeof(v0));
            memcpy(v1, src + s0_s + 4096, sizeof(v1));
            memcpy(v2, src + s0_s + 67108864, sizeof(v2));
            memcpy(v3, src + s0_s + 67112960, sizeof(v3));
            memcpy(v4, src + s0_s + 8, sizeof(v4));
            memcpy(v5, src + s0_s + 4104, sizeof(v5));
            memcpy(v6, src + s0_s + 67108872, sizeof(v6));
            memcpy(v7, src + s0_s + 67112968, sizeof(v7));
            memcpy(v8, src + s1_s + 0, sizeof(v8));
            memcpy(v9, src + s1_s + 4096, sizeof(v9));
            memcpy(v10, src + s1_s + 67108864, sizeof(v10));
            memcpy(v11, src + s1_s + 67112960, sizeof(v11));
            memcpy(v12, src + s1_s + 8, sizeof(v12));
            memcpy(v13, src + s1_s + 4104, sizeof(v13));
            memcpy(v14, src + s1_s + 67108872, sizeof(v14));
            memcpy(v15, src + s1_s + 67112968, sizeof(v15));
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v0[vp_tab0[k]] : v1[vp_tab0[k] - 8]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v0[vp_tab1[k]] : v1[vp_tab1[k] - 8]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v2[vp_tab0[k]] : v3[vp_tab0[k] - 8]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v2[vp_tab1[k]] : v3[vp_tab1[k] - 8]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v4[vp_tab0[k]] : v5[vp_tab0[k] - 8]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v4[vp_tab1[k]] : v5[vp_tab1[k] - 8]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v6[vp_tab0[k]] : v7[vp_tab0[k] - 8]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v6[vp_tab1[k]] : v7[vp_tab1[k] - 8]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v8[vp_tab0[k]] : v9[vp_tab0[k] - 8]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v8[vp_tab1[k]] : v9[vp_tab1[k] - 8]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v10[vp_tab0[k]] : v11[vp_tab0[k] - 8]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v10[vp_tab1[k]] : v11[vp_tab1[k] - 8]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v12[vp_tab0[k]] : v13[vp_tab0[k] - 8]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v12[vp_tab1[k]] : v13[vp_tab1[k] - 8]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab0[k] < 8 ? v14[vp_tab0[k]] : v15[vp_tab0[k] - 8]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab1[k] < 8 ? v14[vp_tab1[k]] : v15[vp_tab1[k] - 8]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v16[vp_tab2[k]] : v0[vp_tab2[k] - 8]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v16[vp_tab3[k]] : v0[vp_tab3[k] - 8]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v17[vp_tab2[k]] : v1[vp_tab2[k] - 8]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v17[vp_tab3[k]] : v1[vp_tab3[k] - 8]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v2[vp_tab2[k]] : v4[vp_tab2[k] - 8]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v2[vp_tab3[k]] : v4[vp_tab3[k] - 8]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v3[vp_tab2[k]] : v5[vp_tab2[k] - 8]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v3[vp_tab3[k]] : v5[vp_tab3[k] - 8]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v14[vp_tab4[k]] : v1[vp_tab4[k] - 8]; memcpy(v3, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v14[vp_tab5[k]] : v1[vp_tab5[k] - 8]; memcpy(v5, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v15[vp_tab4[k]] : v17[vp_tab4[k] - 8]; memcpy(v1, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v15[vp_tab5[k]] : v17[vp_tab5[k] - 8]; memcpy(v14, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v0[vp_tab4[k]] : v2[vp_tab4[k] - 8]; memcpy(v15, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v0[vp_tab5[k]] : v2[vp_tab5[k] - 8]; memcpy(v17, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v16[vp_tab4[k]] : v4[vp_tab4[k] - 8]; memcpy(v0, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v16[vp_tab5[k]] : v4[vp_tab5[k] - 8]; memcpy(v2, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v6[vp_tab2[k]] : v8[vp_tab2[k] - 8]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v6[vp_tab3[k]] : v8[vp_tab3[k] - 8]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v7[vp_tab2[k]] : v9[vp_tab2[k] - 8]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v7[vp_tab3[k]] : v9[vp_tab3[k] - 8]; memcpy(v8, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v10[vp_tab2[k]] : v12[vp_tab2[k] - 8]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v10[vp_tab3[k]] : v12[vp_tab3[k] - 8]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab2[k] < 8 ? v11[vp_tab2[k]] : v13[vp_tab2[k] - 8]; memcpy(v10, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab3[k] < 8 ? v11[vp_tab3[k]] : v13[vp_tab3[k] - 8]; memcpy(v12, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v4[vp_tab4[k]] : v7[vp_tab4[k] - 8]; memcpy(v11, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v4[vp_tab5[k]] : v7[vp_tab5[k] - 8]; memcpy(v13, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v16[vp_tab4[k]] : v9[vp_tab4[k] - 8]; memcpy(v4, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v16[vp_tab5[k]] : v9[vp_tab5[k] - 8]; memcpy(v7, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v6[vp_tab4[k]] : v10[vp_tab4[k] - 8]; memcpy(v9, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v6[vp_tab5[k]] : v10[vp_tab5[k] - 8]; memcpy(v16, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab4[k] < 8 ? v8[vp_tab4[k]] : v12[vp_tab4[k] - 8]; memcpy(v6, vp_t, sizeof(vp_t)); }
            { vp_elem_t vp_t[8]; int k; for (k = 0; k < 8; ++k) vp_t[k] = vp_tab5[k] < 8 ? v8[vp_tab5[k]] : v12[vp_tab5[k] - 8]; memcpy(v10, vp_t, sizeof(vp_t)); }
            memcpy(dst + s0_d + 0, v3, sizeof(v3));
            memcpy(dst + s0_d + 8, v5, sizeof(v5));
            memcpy(dst + s0_d + 2097152, v1, sizeof(v1));
            memcpy(dst + s0_d + 2097160, v14, sizeof(v14));
            memcpy(dst + s0_d + 8388608, v15, sizeof(v15));
            memcpy(dst + s0_d + 8388616, v17, sizeof(v17));
            memcpy(dst + s0_d + 10485760, v0, sizeof(v0));
            memcpy(dst + s0_d + 10485768, v2, sizeof(v2));
            memcpy(dst + s1_d + 0, v11, sizeof(v11));
            memcpy(dst + s1_d + 8, v13, sizeof(v13));
            memcpy(dst + s1_d + 2097152, v4, sizeof(v4));
            memcpy(dst + s1_d + 2097160, v7, sizeof(v7));
            memcpy(dst + s1_d + 8388608, v9, sizeof(v9));
            memcpy(dst + s1_d + 8388616, v16, sizeof(v16));
            memcpy(dst + s1_d + 10485760, v6, sizeof(v6));
            memcpy(dst + s1_d + 10485768, v10, sizeof(v10));
        }
    }
}
