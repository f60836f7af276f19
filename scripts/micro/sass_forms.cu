// How ptxas (CUDA 12.9, sm_100a) lowers the instruction forms the K5b hot loop would
// like to use.  Compile only -- no GPU needed:
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -cubin -o /tmp/f.cubin \
//        scripts/micro/sass_forms.cu && cuobjdump -sass /tmp/f.cubin
//
// Findings (profiles/r2_k5b_sass.md):
//   k_red_*      every predicated reduction (@p red.global.add, f64/f32/u64, volatile or
//                not, .relaxed.gpu or not, with or without a "memory" clobber) becomes
//                BSSY / @!P BRA / REDG / BSYNC; sm_90a does the same.
//   k_st         a predicated store stays one @P STG (the branch is RED-specific).
//   k_padd       @p add.rn.f64 is if-converted into an unconditional DADD + 2 FSEL (the
//                masked fma of dda_advance is one DFMA + 1 FSEL + 1 zero move instead).
//   k_fmin       fmin(double) is DSETP.MIN + FSEL + SEL + @P LOP3 (NaN quieting): more
//                than the DSETP + 2 FSEL of `c ? a : b`.

__device__ __forceinline__ void red_v(bool e, double* a, double x) {
    asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p red.global.add.f64 [%1], %2;}"
                 ::"r"((int)e), "l"(a), "d"(x) : "memory");
}
__device__ __forceinline__ void red_relaxed(bool e, double* a, double x) {
    asm("{.reg .pred p; setp.ne.b32 p, %0, 0; @p red.relaxed.gpu.global.add.f64 [%1], %2;}"
        ::"r"((int)e), "l"(a), "d"(x));
}

__global__ void k_red_f64(double* g, const int* idx, const double* v, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int a = idx[j];
        const double x = v[j];
        red_v(a & 1, g + a, x);
        red_v(a & 2, g + a + 1, 2 * x);
    }
}
__global__ void k_red_relaxed(double* g, const int* idx, const double* v, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int a = idx[j];
        const double x = v[j];
        red_relaxed(a & 1, g + a, x);
        red_relaxed(a & 2, g + a + 1, 2 * x);
    }
}
__global__ void k_red_f32(float* g, const int* idx, const float* v, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int a = idx[j];
        asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p red.global.add.f32 [%1], %2;}"
                     ::"r"(a & 1), "l"(g + a), "f"(v[j]) : "memory");
    }
}
__global__ void k_red_u64(unsigned long long* g, const int* idx, const unsigned long long* v, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int a = idx[j];
        asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p red.global.add.u64 [%1], %2;}"
                     ::"r"(a & 1), "l"(g + a), "l"(v[j]) : "memory");
    }
}
__global__ void k_st(double* g, const int* idx, const double* v, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const int a = idx[j];
        asm volatile("{.reg .pred p; setp.ne.b32 p, %0, 0; @p st.global.f64 [%1], %2;}"
                     ::"r"(a & 1), "l"(g + a), "d"(v[j]) : "memory");
    }
}

// One DDA advance written with predicated adds and with fmin.
__global__ void k_padd(double* out, const double* in, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double tx = in[i], ty = in[i + n], tz = in[i + 2 * n];
    const double dx = in[i + 3 * n], dy = in[i + 4 * n], dz = in[i + 5 * n], t1 = in[i + 6 * n];
    double acc = 0.0, t = 0.0;
    for (;;) {
        const bool c1 = ty < tx;
        const double m01 = c1 ? ty : tx;
        const bool c2 = tz < m01;
        const double tm = c2 ? tz : m01;
        const int a0 = !c2 && !c1, a1 = !c2 && c1, a2 = c2;
        asm("{.reg .pred q0, q1, q2;\n\t"
            "setp.ne.b32 q0, %3, 0; setp.ne.b32 q1, %4, 0; setp.ne.b32 q2, %5, 0;\n\t"
            "@q0 add.rn.f64 %0, %0, %6;\n\t@q1 add.rn.f64 %1, %1, %7;\n\t@q2 add.rn.f64 %2, %2, %8;}"
            : "+d"(tx), "+d"(ty), "+d"(tz)
            : "r"(a0), "r"(a1), "r"(a2), "d"(dx), "d"(dy), "d"(dz));
        acc += tm - t;
        t = tm;
        if (tm >= t1) break;
    }
    out[i] = acc;
}
__global__ void k_fmin(double* out, const double* in, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    out[i] = fmin(fmin(in[i], in[i + n]), in[i + 2 * n]);
}
