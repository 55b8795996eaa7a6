// n1_interp_bench.cu -- cost of SURVEY.md §8(f) N1 (frequency-space rotation, PAPER.md L271
// "the rotations are handled by an interpolation over the frequency grid") on the sweep's
// band: per rotation, B_hat(R^T k) for every band mode k (M x M x Kz = 511 x 511 x 256 real-
// weight half band) interpolated from a table of B_hat tabulated once on an oversampled
// lattice, with a separable width-w Kaiser-Bessel kernel (w^3 taps per mode).
//
// B's support radius rho_B = 0.22 (sweep) makes B_hat band-limited in the frequency variable:
// a lattice spacing d_xi <= 1 / (2 rho_B sigma) with oversampling sigma suffices.  With the
// band's |xi| <= sqrt(3) 255 / P (P = 2), sigma = 1.25 gives 245 samples per axis: a
// 245^3 complex64 table = 118 MB, L2-resident on B200 (126 MB) -- the best case for N1.
// The kernel reads the table through L2 (random-ish gathers), evaluates the separable KB
// weights in registers and accumulates w^3 products; its time per rotation is what N1 would
// cost before the product / fold / inverse FFT it shares with the current path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/n1 tools/n1_interp_bench.cu && /tmp/n1
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

constexpr int TB = 245;              // table points per axis
constexpr int KB = 255, M = 2 * KB + 1, KZ = KB + 1;

template <int W>
__global__ void __launch_bounds__(256) interp_kernel(const float2 *__restrict__ tab, const float *R, float scale,
                                                     float beta, float2 *out, long long n)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int kx = (int)(e % M) - KB, ky = (int)((e / M) % M) - KB, kz = (int)(e / ((long long)M * M));
    // R^T k in table units (table centre at TB / 2)
    const float u[3] = {(R[0] * kx + R[3] * ky + R[6] * kz) * scale + TB / 2,
                        (R[1] * kx + R[4] * ky + R[7] * kz) * scale + TB / 2,
                        (R[2] * kx + R[5] * ky + R[8] * kz) * scale + TB / 2};
    int i0[3];
    float w[3][W];
#pragma unroll
    for (int d = 0; d < 3; d++) {
        i0[d] = (int)floorf(u[d]) - W / 2 + 1;
#pragma unroll
        for (int q = 0; q < W; q++) {
            const float x = (u[d] - (float)(i0[d] + q)) * (2.f / W);
            const float a = fmaxf(1.f - x * x, 0.f);
            w[d][q] = __expf(beta * (sqrtf(a) - 1.f));  // KB-like window (exp form)
        }
    }
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int a = 0; a < W; a++)
#pragma unroll
        for (int b = 0; b < W; b++) {
            const float wab = w[0][a] * w[1][b];
            const float2 *row = tab + ((long long)(i0[0] + a) * TB + (i0[1] + b)) * TB + i0[2];
#pragma unroll
            for (int c = 0; c < W; c++) {
                const float2 t = __ldg(row + c);
                acc.x += wab * w[2][c] * t.x;
                acc.y += wab * w[2][c] * t.y;
            }
        }
    out[e] = acc;
}

template <int W>
float run(const float2 *tab, const float *R, float2 *out, long long n)
{
    const float scale = (float)(TB - 2 * W - 2) / (2.f * 1.7320508f * KB);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const unsigned g = (unsigned)((n + 255) / 256);
    for (int i = 0; i < 3; i++) interp_kernel<W><<<g, 256>>>(tab, R, scale, 2.3f * W, out, n);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int i = 0; i < reps; i++) interp_kernel<W><<<g, 256>>>(tab, R, scale, 2.3f * W, out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

int main()
{
    const long long n = (long long)M * M * KZ;  // half band of the sweep (real weights)
    const size_t tb = (size_t)TB * TB * TB;
    float2 *tab, *out;
    float *R;
    cudaMalloc(&tab, tb * sizeof(float2));
    cudaMalloc(&out, n * sizeof(float2));
    cudaMalloc(&R, 9 * sizeof(float));
    cudaMemset(tab, 0, tb * sizeof(float2));
    const float c = 0.8f, s = 0.6f;  // a generic rotation (about z then the mixing below)
    const float hR[9] = {c, -s, 0.f, s * 0.8f, c * 0.8f, -0.6f, s * 0.6f, c * 0.6f, 0.8f};
    cudaMemcpy(R, hR, sizeof(hR), cudaMemcpyHostToDevice);
    const float t2 = run<2>(tab, R, out, n), t4 = run<4>(tab, R, out, n), t6 = run<6>(tab, R, out, n);
    const cudaError_t err = cudaGetLastError();
    printf("{\"modes_per_rotation\": %lld, \"table_MB\": %.1f, \"ms_per_rotation\": {\"w2\": %.4f, \"w4\": %.4f, "
           "\"w6\": %.4f}, \"cuda\": \"%s\"}\n",
           n, tb * 8 / 1e6, t2, t4, t6, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
