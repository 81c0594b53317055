// init.cuh — on-device random-init weights from the counter hash in
// include/cascade_weights.h, written straight into the layouts the kernels
// consume (A-frag for streamed matrices, row-major for embedding, router
// and norms).  Nothing crosses PCIe; the oracle regenerates any element.
#pragma once

#include "common.cuh"
#include "gemv_umma.cuh"

namespace cascade {

enum RowMap : int {
    ROWMAP_SIMPLE = 0,   // phys row r -> (kind0, r)
    ROWMAP_GATEUP = 1,   // 16-row tile i: rows 0-7 gate[8i..8i+7], rows 8-15 up[8i..]
    ROWMAP_QKV = 2,      // [0,n0) kind0, [n0,n0+n1) kind1, rest kind2
};

struct InitParams {
    uint4* dst;          // A-frag storage
    long long n_vec;     // number of uint4 (8 bf16) in the tensor
    int n_ks;            // K / 16
    int rowmap;
    int n0, n1;          // ROWMAP_QKV split
    uint64_t key[3];     // per logical kind
    float scale[3];
    int cols;            // logical K (row stride of the hashed index)
    int umma;            // 1: UMMA A layout (gemv_umma.cuh), 0: A-frag (gemv.cuh)
};

__global__ void init_afrag_kernel(InitParams p) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < p.n_vec;
         q += (long long)gridDim.x * blockDim.x) {
        const int lane = (int)(q & 31);
        const long long q2 = q >> 5;
        const int it = (int)(q2 % kTPW);
        const long long q3 = q2 / kTPW;
        const int s = (int)(q3 % p.n_ks);
        const long long st = q3 / p.n_ks;
        // UMMA layout: uint4 q = 8 consecutive columns of one row of a core matrix
        const long long ku = q % ((long long)p.n_ks * 2 * kURows);
        const long long unit = q / ((long long)p.n_ks * 2 * kURows);
        const int us = (int)(ku / (2 * kURows)), ukc = (int)((ku / kURows) & 1), ur = (int)(ku % kURows);
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
            uint16_t v[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                long long prow;
                int col;
                if (p.umma) {
                    prow = unit * kURows + ur;
                    col = us * 16 + ukc * 8 + e + h;
                } else {
                    int r, c;
                    afrag_coords(lane, e + h, r, c);
                    prow = st * kSTRows + it * 16 + r;
                    col = s * 16 + c;
                }
                int kind = 0;
                long long lrow = prow;
                if (p.rowmap == ROWMAP_GATEUP) {
                    const long long tile = prow >> 4;
                    const int r16 = (int)(prow & 15);
                    kind = r16 < 8 ? 0 : 1;
                    lrow = tile * 8 + (r16 & 7);
                } else if (p.rowmap == ROWMAP_QKV) {
                    if (prow < p.n0) {
                        kind = 0;
                    } else if (prow < p.n0 + p.n1) {
                        kind = 1;
                        lrow = prow - p.n0;
                    } else {
                        kind = 2;
                        lrow = prow - p.n0 - p.n1;
                    }
                }
                v[h] = cascade_weight_bits(p.key[kind], (uint64_t)lrow * p.cols + col, p.scale[kind]);
            }
            w[e / 2] = (uint32_t)v[0] | ((uint32_t)v[1] << 16);
        }
        p.dst[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Row-major [rows][cols] bf16; rows >= valid_rows are zero (router padding).
__global__ void init_plain_kernel(uint16_t* dst, long long n, int cols, long long valid,
                                  uint64_t key, float scale, long long row_offset) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols + row_offset;
        const int c = (int)(i % cols);
        dst[i] = i < valid ? cascade_weight_bits(key, (uint64_t)r * cols + c, scale) : (uint16_t)0;
    }
}

}  // namespace cascade
