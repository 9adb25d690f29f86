// K10: EvictionNet training on the GPU (net.py:107-279).
//
// The reference trains one net per layer (cli.py:253-283), each a float64
// numpy loop of mini-batch forward / backward / AdamW steps.  Here every
// layer's net trains at once: one mcb_train_epoch call runs all mini-batches
// of one epoch for all nets, the GEMMs as strided-batched cuBLAS DGEMMs over
// the nets (plain library GEMMs on the fp64 tensor cores), everything else
// in the kernels below:
//   k_gather        mini-batch rows by the epoch's permutation (features,
//                   targets, masks of every net)
//   k_bias_silu     z += b; h = silu(z) with the reference's sign-split
//                   logistic (net.py:43-55)
//   k_mse_grad      per net: masked MSE of the batch and dLoss/dOut
//                   (net.py:141-156), non-finite loss recorded
//   k_silu_back     dz = dh * silu'(z)
//   k_colsum        bias gradients (column sums over the batch)
//   k_adamw         decoupled-weight-decay Adam (net.py:159-184)
// AdamW, the loss gradient and the activations use the reference's
// operation order without FMA contraction, so they are exact given their
// inputs; GEMM summation order (and exp's last ulp) differ from numpy's BLAS,
// so parity with the reference trainer is to a tolerance
// (tests/test_train_gpu.py).  Reductions are ordered (no float atomics), so
// training is deterministic run to run.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mcb_internal.h"

namespace train {

__device__ __forceinline__ double sigmoid_ref(double z) {   // net.py:43-49
    if (z >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
    const double ez = exp(z);
    return __ddiv_rn(ez, __dadd_rn(1.0, ez));
}

__global__ void k_gather(int E, int64_t n, int B, int64_t start, const int32_t *__restrict__ order,
                         const double *__restrict__ feat, const double *__restrict__ targ,
                         const uint8_t *__restrict__ mask, double *xb, double *yb, double *mb) {
    const int net = blockIdx.y;
    const int r = blockIdx.x;
    const int64_t row = order[start + r];
    const double *f = feat + ((int64_t)net * n + row) * 2 * E;
    const double *t = targ + ((int64_t)net * n + row) * E;
    const uint8_t *m = mask + ((int64_t)net * n + row) * E;
    double *xo = xb + ((int64_t)net * B + r) * 2 * E;
    double *yo = yb + ((int64_t)net * B + r) * E;
    double *mo = mb + ((int64_t)net * B + r) * E;
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) xo[i] = f[i];
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
        yo[i] = t[i];
        mo[i] = m[i] ? 1.0 : 0.0;
    }
}

// z[net][r][j] += b[net][j]; h = z * sigmoid(z)
__global__ void k_bias_silu(int64_t rows, int H, int64_t z_stride, int64_t b_stride, double *z,
                            const double *b, double *h) {
    const int net = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * H) return;
    const int j = (int)(i % H);
    double *zz = z + net * z_stride;
    const double v = __dadd_rn(zz[i], b[net * b_stride + j]);
    zz[i] = v;
    if (h) h[net * z_stride + i] = __dmul_rn(v, sigmoid_ref(v));
}

// out += b3 (linear output)
__global__ void k_bias(int64_t rows, int E, int64_t o_stride, int64_t b_stride, double *o, const double *b) {
    const int net = blockIdx.y;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * E) return;
    o[net * o_stride + i] = __dadd_rn(o[net * o_stride + i], b[net * b_stride + (int)(i % E)]);
}

// One block per net: masked MSE of the batch (net.py:141-147) and the loss
// gradient 2 m (pred - y) / denom (net.py:150-156) written over `pred`.
// bad[net] = {flag, loss, batch offset} of the first non-finite loss.
__global__ void __launch_bounds__(256) k_mse_grad(int rows, int E, int64_t stride, double *pred, const double *yb,
                                                  const double *mb, double *bad, int64_t start, int64_t epoch) {
    const int net = blockIdx.x;
    const int64_t n = (int64_t)rows * E;
    double *p = pred + net * stride;
    const double *y = yb + net * stride;
    const double *m = mb + net * stride;
    __shared__ double s_num[256], s_den[256];
    double num = 0.0, den = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = __dsub_rn(p[i], y[i]);
        num = __dadd_rn(num, __dmul_rn(m[i], __dmul_rn(d, d)));
        den = __dadd_rn(den, m[i]);
    }
    s_num[threadIdx.x] = num;
    s_den[threadIdx.x] = den;
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        if ((int)threadIdx.x < w) {
            s_num[threadIdx.x] = __dadd_rn(s_num[threadIdx.x], s_num[threadIdx.x + w]);
            s_den[threadIdx.x] = __dadd_rn(s_den[threadIdx.x], s_den[threadIdx.x + w]);
        }
        __syncthreads();
    }
    const double tot = s_den[0];
    const double loss = tot == 0.0 ? 0.0 : __ddiv_rn(s_num[0], tot);
    if (threadIdx.x == 0 && !isfinite(loss) && bad[net * 4] == 0.0) {
        bad[net * 4 + 0] = 1.0;
        bad[net * 4 + 1] = loss;
        bad[net * 4 + 2] = (double)start;
        bad[net * 4 + 3] = (double)epoch;
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
        p[i] = tot == 0.0 ? 0.0 : __ddiv_rn(__dmul_rn(__dmul_rn(2.0, m[i]), __dsub_rn(p[i], y[i])), tot);
}

// dz = dh * s * (1 + z * (1 - s)), s = sigmoid(z)   (silu_grad, net.py:56-58)
__global__ void k_silu_back(int64_t count, double *dh, const double *z) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double zz = z[i];
    const double s = sigmoid_ref(zz);
    const double g = __dmul_rn(s, __dadd_rn(1.0, __dmul_rn(zz, __dsub_rn(1.0, s))));
    dh[i] = __dmul_rn(dh[i], g);
}

// g[net][j] = sum_r d[net][r][j]  (row order)
__global__ void k_colsum(int rows, int cols, int64_t d_stride, const double *d, int64_t g_stride, double *g) {
    const int net = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= cols) return;
    const double *dd = d + net * d_stride;
    double acc = 0.0;
    for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, dd[(int64_t)r * cols + j]);
    g[net * g_stride + j] = acc;
}

// AdamW.step (net.py:172-184), element-wise over every parameter of every net
__global__ void k_adamw(int64_t count, double *p, const double *g, double *m, double *v, double lr, double wd,
                        double b1, double b2, double eps, double b1c, double b2c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const double gi = g[i];
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), gi));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, b1c);
    const double vh = __ddiv_rn(vi, b2c);
    const double pi = p[i];
    const double upd = __dadd_rn(__ddiv_rn(mh, __dadd_rn(__dsqrt_rn(vh), eps)), __dmul_rn(wd, pi));
    p[i] = __dsub_rn(pi, __dmul_rn(lr, upd));
}

// per (net, block) partial sums of m * (pred - y)^2 and m over a row range
__global__ void __launch_bounds__(256) k_mse_partial(int64_t rows, int E, const double *pred, int64_t p_stride,
                                                     const double *targ, const uint8_t *mask, int64_t n,
                                                     int64_t row0, double *part) {
    const int net = blockIdx.y;
    const int64_t cnt = rows * E;
    const double *p = pred + net * p_stride;
    const double *y = targ + ((int64_t)net * n + row0) * E;
    const uint8_t *mk = mask + ((int64_t)net * n + row0) * E;
    __shared__ double s_num[256], s_den[256];
    double num = 0.0, den = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
        const double m = mk[i] ? 1.0 : 0.0;   // m * (pred - target) ** 2, NaN-propagating like numpy
        const double d = __dsub_rn(p[i], y[i]);
        num = __dadd_rn(num, __dmul_rn(m, __dmul_rn(d, d)));
        den = __dadd_rn(den, m);
    }
    s_num[threadIdx.x] = num;
    s_den[threadIdx.x] = den;
    __syncthreads();
    for (int w = 128; w >= 1; w >>= 1) {
        if ((int)threadIdx.x < w) {
            s_num[threadIdx.x] = __dadd_rn(s_num[threadIdx.x], s_num[threadIdx.x + w]);
            s_den[threadIdx.x] = __dadd_rn(s_den[threadIdx.x], s_den[threadIdx.x + w]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[((int64_t)net * gridDim.x + blockIdx.x) * 2 + 0] = s_num[0];
        part[((int64_t)net * gridDim.x + blockIdx.x) * 2 + 1] = s_den[0];
    }
}

__global__ void k_mse_final(int n_nets, int blocks, const double *part, double *sums) {
    const int net = blockIdx.x * blockDim.x + threadIdx.x;
    if (net >= n_nets) return;
    double a = sums[net * 2], b = sums[net * 2 + 1];
    for (int k = 0; k < blocks; ++k) {
        a = __dadd_rn(a, part[((int64_t)net * blocks + k) * 2]);
        b = __dadd_rn(b, part[((int64_t)net * blocks + k) * 2 + 1]);
    }
    sums[net * 2] = a;
    sums[net * 2 + 1] = b;
}

}  // namespace train

// ---------------------------------------------------------------- host side --

int mcb_ctx_scratch_named(mcb_ctx *c, int slot, size_t bytes, void **p);   // mcb_api.cu
cublasHandle_t mcb_ctx_cublas(mcb_ctx *c);                                // mcb_api.cu

namespace {

struct Shapes {
    int N, E, H;
    int64_t P;            // parameters per net
    int64_t o_w1, o_b1, o_w2, o_b2, o_w3, o_b3;
};

Shapes shapes_of(const mcb_train_data *d) {
    Shapes s;
    s.N = d->num_nets;
    s.E = d->num_experts;
    s.H = d->hidden;
    const int64_t E = s.E, H = s.H;
    s.o_w1 = 0;
    s.o_b1 = s.o_w1 + H * 2 * E;
    s.o_w2 = s.o_b1 + H;
    s.o_b2 = s.o_w2 + H * H;
    s.o_w3 = s.o_b2 + H;
    s.o_b3 = s.o_w3 + E * H;
    s.P = s.o_b3 + E;
    return s;
}

// Row-major C[M][N] (+)= op(A) op(B) for `batch` nets (cuBLAS is column-major:
// C^T = op(B)^T op(A)^T).  ta / tb: the row-major operand is transposed.
cublasStatus_t rm_gemm(cublasHandle_t h, bool ta, bool tb, int M, int N, int K, const double *A, int lda,
                       long long sA, const double *B, int ldb, long long sB, double beta, double *C, int ldc,
                       long long sC, int batch) {
    const double one = 1.0;
    return cublasDgemmStridedBatched(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, N, M, K,
                                     &one, B, ldb, sB, A, lda, sA, &beta, C, ldc, sC, batch);
}

struct Work {
    double *xb, *yb, *mb, *z1, *h1, *z2, *h2, *out, *dh, *grad;
};

int forward(cublasHandle_t h, const Shapes &S, const double *params, const double *x, int64_t x_stride, int rows,
            double *z1, double *h1, double *z2, double *h2, double *out, int64_t hs, int64_t os, cudaStream_t st) {
    const int E = S.E, H = S.H, N = S.N;
    const long long sp = S.P;
    const unsigned gh = (unsigned)(((int64_t)rows * H + 255) / 256), go = (unsigned)(((int64_t)rows * E + 255) / 256);
    // z1 = x w1^T
    if (rm_gemm(h, false, true, rows, H, 2 * E, x, 2 * E, x_stride, params + S.o_w1, 2 * E, sp, 0.0, z1, H, hs, N))
        return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
    train::k_bias_silu<<<dim3(gh, N), 256, 0, st>>>(rows, H, hs, S.P, z1, params + S.o_b1, h1);
    if (rm_gemm(h, false, true, rows, H, H, h1, H, hs, params + S.o_w2, H, sp, 0.0, z2, H, hs, N))
        return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
    train::k_bias_silu<<<dim3(gh, N), 256, 0, st>>>(rows, H, hs, S.P, z2, params + S.o_b2, h2);
    if (rm_gemm(h, false, true, rows, E, H, h2, H, hs, params + S.o_w3, H, sp, 0.0, out, E, os, N))
        return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
    train::k_bias<<<dim3(go, N), 256, 0, st>>>(rows, E, os, S.P, out, params + S.o_b3);
    return MCB_OK;
}

int check_data(const mcb_train_data *d) {
    if (!d || !d->features || !d->targets || !d->masks) return mcb_set_error(MCB_ERR_INVALID, "NULL training data");
    if (d->num_nets < 1 || d->num_experts < 1 || d->hidden < 1 || d->num_samples < 1)
        return mcb_set_error(MCB_ERR_INVALID, "invalid training shapes");
    return MCB_OK;
}

}  // namespace

extern "C" int mcb_train_epoch(mcb_ctx *ctx, const mcb_train_data *data, const mcb_train_cfg *cfg, double *params,
                               double *adam_m, double *adam_v, int64_t step0, int64_t epoch, const int32_t *order,
                               double *bad, void *stream) {
    mcb_clear_error();
    if (!ctx) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_data(data)) return rc;
    if (!cfg || !params || !adam_m || !adam_v || !order || !bad) return mcb_set_error(MCB_ERR_INVALID, "NULL pointer");
    if (cfg->batch_size < 1 || cfg->n_train < 1 || cfg->n_train > data->num_samples)
        return mcb_set_error(MCB_ERR_INVALID, "invalid batch_size / n_train");
    const Shapes S = shapes_of(data);
    const int B = (int)(cfg->batch_size < cfg->n_train ? cfg->batch_size : cfg->n_train);
    const int E = S.E, H = S.H, N = S.N;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nb = (int64_t)N * B;
    const size_t words = (size_t)nb * (2 * E + E + E + 4 * H + E + H) + (size_t)N * S.P;
    void *wp = nullptr;
    if (int rc = mcb_ctx_scratch_named(ctx, 0, words * sizeof(double), &wp)) return rc;
    Work w;
    w.xb = (double *)wp;
    w.yb = w.xb + nb * 2 * E;
    w.mb = w.yb + nb * E;
    w.z1 = w.mb + nb * E;
    w.h1 = w.z1 + nb * H;
    w.z2 = w.h1 + nb * H;
    w.h2 = w.z2 + nb * H;
    w.out = w.h2 + nb * H;
    w.dh = w.out + nb * E;
    w.grad = w.dh + nb * H;
    cublasHandle_t h = mcb_ctx_cublas(ctx);
    if (!h) return mcb_set_error(MCB_ERR_CUDA, "cublasCreate failed");
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return mcb_set_error(MCB_ERR_CUDA, "cublasSetStream failed");
    const long long sp = S.P, sx = (long long)B * 2 * E, sh = (long long)B * H, so = (long long)B * E;
    int64_t t = step0;
    for (int64_t start = 0; start < cfg->n_train; start += cfg->batch_size) {
        const int rows = (int)((cfg->n_train - start) < cfg->batch_size ? (cfg->n_train - start) : cfg->batch_size);
        train::k_gather<<<dim3(rows, N), 64, 0, st>>>(E, data->num_samples, B, start, order, data->features,
                                                      data->targets, data->masks, w.xb, w.yb, w.mb);
        if (int rc = forward(h, S, params, w.xb, sx, rows, w.z1, w.h1, w.z2, w.h2, w.out, sh, so, st)) return rc;
        // masked-MSE gradient (written over out) on a dense [rows][E] block per net
        train::k_mse_grad<<<N, 256, 0, st>>>(rows, E, so, w.out, w.yb, w.mb, bad, start, epoch);
        double *g = w.grad;
        // w3 / b3
        if (rm_gemm(h, true, false, E, H, rows, w.out, E, so, w.h2, H, sh, 0.0, g + S.o_w3, H, sp, N))
            return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
        train::k_colsum<<<dim3((E + 127) / 128, N), 128, 0, st>>>(rows, E, so, w.out, S.P, g + S.o_b3);
        // dh2 = dout w3 ; dz2
        if (rm_gemm(h, false, false, rows, H, E, w.out, E, so, params + S.o_w3, H, sp, 0.0, w.dh, H, sh, N))
            return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
        train::k_silu_back<<<(unsigned)((nb * H + 255) / 256), 256, 0, st>>>(nb * H, w.dh, w.z2);
        if (rm_gemm(h, true, false, H, H, rows, w.dh, H, sh, w.h1, H, sh, 0.0, g + S.o_w2, H, sp, N))
            return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
        train::k_colsum<<<dim3((H + 127) / 128, N), 128, 0, st>>>(rows, H, sh, w.dh, S.P, g + S.o_b2);
        // dh1 = dz2 w2 (into h2's buffer, free now) ; dz1
        if (rm_gemm(h, false, false, rows, H, H, w.dh, H, sh, params + S.o_w2, H, sp, 0.0, w.h2, H, sh, N))
            return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
        train::k_silu_back<<<(unsigned)((nb * H + 255) / 256), 256, 0, st>>>(nb * H, w.h2, w.z1);
        if (rm_gemm(h, true, false, H, 2 * E, rows, w.h2, H, sh, w.xb, 2 * E, sx, 0.0, g + S.o_w1, 2 * E, sp, N))
            return mcb_set_error(MCB_ERR_CUDA, "cublasDgemmStridedBatched failed");
        train::k_colsum<<<dim3((H + 127) / 128, N), 128, 0, st>>>(rows, H, sh, w.h2, S.P, g + S.o_b1);
        ++t;
        const double b1c = 1.0 - pow(cfg->beta1, (double)t), b2c = 1.0 - pow(cfg->beta2, (double)t);
        const int64_t cnt = (int64_t)N * S.P;
        train::k_adamw<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(cnt, params, g, adam_m, adam_v,
                                                                      cfg->learning_rate, cfg->weight_decay,
                                                                      cfg->beta1, cfg->beta2, cfg->eps, b1c, b2c);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}

extern "C" int mcb_train_eval(mcb_ctx *ctx, const mcb_train_data *data, const double *params, int64_t row0,
                              int64_t rows, double *sums, void *stream) {
    mcb_clear_error();
    if (!ctx) return mcb_set_error(MCB_ERR_INVALID, "ctx is NULL");
    if (int rc = check_data(data)) return rc;
    if (!params || !sums) return mcb_set_error(MCB_ERR_INVALID, "NULL pointer");
    if (row0 < 0 || rows < 0 || row0 + rows > data->num_samples)
        return mcb_set_error(MCB_ERR_INVALID, "row range outside the dataset");
    const Shapes S = shapes_of(data);
    const int E = S.E, H = S.H, N = S.N;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(sums, 0, (size_t)N * 2 * sizeof(double), st);
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    if (rows == 0) return MCB_OK;
    const int64_t chunk = rows < 8192 ? rows : 8192;
    const int part_blocks = 64;
    const size_t words = (size_t)N * chunk * (4 * H + E) + (size_t)N * part_blocks * 2;
    void *wp = nullptr;
    if (int rc = mcb_ctx_scratch_named(ctx, 1, words * sizeof(double), &wp)) return rc;
    double *z1 = (double *)wp, *h1 = z1 + N * chunk * H, *z2 = h1 + N * chunk * H, *h2 = z2 + N * chunk * H;
    double *out = h2 + N * chunk * H, *part = out + N * chunk * E;
    cublasHandle_t h = mcb_ctx_cublas(ctx);
    if (!h) return mcb_set_error(MCB_ERR_CUDA, "cublasCreate failed");
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return mcb_set_error(MCB_ERR_CUDA, "cublasSetStream failed");
    for (int64_t r = row0; r < row0 + rows; r += chunk) {
        const int n = (int)((row0 + rows - r) < chunk ? (row0 + rows - r) : chunk);
        const double *x = data->features + r * 2 * E;   // net stride = num_samples * 2E
        if (int rc = forward(h, S, params, x, data->num_samples * 2 * E, n, z1, h1, z2, h2, out,
                             (long long)chunk * H, (long long)chunk * E, st))
            return rc;
        train::k_mse_partial<<<dim3(part_blocks, N), 256, 0, st>>>(n, E, out, chunk * E, data->targets, data->masks,
                                                                   data->num_samples, r, part);
        train::k_mse_final<<<(N + 127) / 128, 128, 0, st>>>(N, part_blocks, part, sums);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return mcb_set_error(MCB_ERR_CUDA, cudaGetErrorString(e));
    return MCB_OK;
}
