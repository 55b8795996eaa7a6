// validate.cu -- on-device validation and conversion of caller arrays that live on the GPU.
//
// bc_correlate_rotations / bc_evaluate_points accept R (and t) in device memory and promise
// to stay asynchronous on the caller's stream (include/ballcorr.h).  Instead of copying the
// arrays to the host to validate them, this kernel checks them where they are -- finite
// entries, R R^T = I within the context's tolerance, det R > 0 (the
// motions are rigid, R in SO(3)) -- writes the fp32 / fp64 copies the path consumes, and
// records a violation in a status word in mapped pinned host memory.  The library reports
// it as BC_EINVAL at the next call or bc_sync on that context (deferred, like an
// asynchronous CUDA fault).
#include "kernels.cuh"

__global__ void rot_prep_kernel(RotPrepArgs a)
{
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= a.n) return;
    double m[9];
    unsigned bad = 0;
#pragma unroll
    for (int q = 0; q < 9; q++) {
        m[q] = a.R[9 * r + q];
        if (!isfinite(m[q])) bad |= BC_DEFER_NONFINITE_R;
    }
    if (!bad) {
#pragma unroll
        for (int i = 0; i < 3; i++)
#pragma unroll
            for (int j = 0; j < 3; j++) {
                const double d = m[3 * i] * m[3 * j] + m[3 * i + 1] * m[3 * j + 1] + m[3 * i + 2] * m[3 * j + 2];
                if (fabs(d - (i == j ? 1.0 : 0.0)) > a.tol) bad |= BC_DEFER_NOT_ORTHONORMAL;
            }
        const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                           m[2] * (m[3] * m[7] - m[4] * m[6]);
        if (!(det > 0)) bad |= BC_DEFER_DET;
    }
    if (a.t) {
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const double v = a.t[3 * r + q];
            if (!isfinite(v)) bad |= BC_DEFER_NONFINITE_T;
            if (a.t64) a.t64[3 * r + q] = v;
        }
    }
#pragma unroll
    for (int q = 0; q < 9; q++) {
        if (a.r32) a.r32[9 * r + q] = (float)m[q];
        if (a.r64) a.r64[9 * r + q] = m[q];
    }
    if (bad) {
        atomicOr(&a.status[0], bad);
        atomicMin(&a.status[1], (unsigned)(a.index_base + r));
        __threadfence_system();
    }
}

void launch_rot_prep(const RotPrepArgs &a, cudaStream_t s)
{
    if (a.n <= 0) return;
    rot_prep_kernel<<<(unsigned)((a.n + 127) / 128), 128, 0, s>>>(a);
}
