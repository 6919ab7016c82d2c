// gen.cu — device twin of synth/__init__.py's counter-based point generator.
// Holds none of CudaPre's arithmetic: it only produces input bytes.  Every
// value is the same fixed sequence of IEEE round-to-nearest operations as the
// numpy implementation (explicit __*_rn intrinsics, no FMA, own log series),
// so both write identical bytes (tests/test_gpu_parity.py checks samples).
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;
constexpr unsigned long long kM1 = 0xBF58476D1CE4E5B9ull;
constexpr unsigned long long kM2 = 0x94D049BB133111EBull;
constexpr unsigned long long kSalt = 0x632BE59BD9B4E019ull;
constexpr int kMaxAttempts = 64;

__host__ __device__ inline unsigned long long mix64(unsigned long long z) {
    z ^= z >> 30;
    z *= kM1;
    z ^= z >> 27;
    z *= kM2;
    return z ^ (z >> 31);
}

__device__ inline unsigned long long draw(unsigned long long key, unsigned long long i, int attempt,
                                          int stream) {
    const unsigned long long ctr = (i << 7) | (unsigned long long)((attempt << 1) | stream);
    return mix64(key + (ctr + 1ull) * kGolden);
}

__device__ inline float u_hi(unsigned long long z) { return __fmul_rn((float)(unsigned)(z >> 40), 0x1p-24f); }
__device__ inline float u_lo(unsigned long long z) {
    return __fmul_rn((float)(unsigned)((z >> 16) & 0xFFFFFFull), 0x1p-24f);
}
__device__ inline float pm1(float u) { return __fsub_rn(__fmul_rn(u, 2.0f), 1.0f); }

__constant__ double kLogCoef[10] = {
    0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5};

__device__ inline double rn_log(double s) {
    int e;
    double m = frexp(s, &e);   // exact: s = m 2^e, m in [0.5, 1)
    if (m < 0x1.6a09e667f3bcdp-1) {
        m = __dmul_rn(m, 2.0);
        e -= 1;
    }
    const double t = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
    const double t2 = __dmul_rn(t, t);
    double p = kLogCoef[9];
    for (int j = 8; j >= 0; --j) {
        p = __dmul_rn(p, t2);
        p = __dadd_rn(p, kLogCoef[j]);
    }
    double lm = __dmul_rn(t, p);
    lm = __dmul_rn(lm, 2.0);
    return __dadd_rn(__dmul_rn((double)e, 0x1.62e42fefa39efp-1), lm);
}

__global__ void gen_kernel(int family, long long n, unsigned long long key, long long base, float lo,
                           float w, double eps, float2* out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const unsigned long long i = (unsigned long long)(base + j);
        float2 r = make_float2(0.f, 0.f);
        if (family == 0) {   // square
            const unsigned long long z = draw(key, i, 0, 0);
            r.x = __fadd_rn(__fmul_rn(u_hi(z), w), lo);
            r.y = __fadd_rn(__fmul_rn(u_lo(z), w), lo);
        } else {
            for (int a = 0; a < kMaxAttempts; ++a) {
                const unsigned long long z = draw(key, i, a, 0);
                const float x = pm1(u_hi(z)), y = pm1(u_lo(z));
                const float s = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
                if (family == 1) {   // disk
                    if (s <= 1.0f) {
                        r = make_float2(x, y);
                        break;
                    }
                } else if (family == 2) {   // gauss (Marsaglia polar)
                    if (s > 0.0f && s < 1.0f) {
                        const double sd = (double)s;
                        const double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(rn_log(sd), -2.0), sd));
                        r.x = __double2float_rn(__dmul_rn((double)x, f));
                        r.y = __double2float_rn(__dmul_rn((double)y, f));
                        break;
                    }
                } else {   // circle: direction of a disk sample, radius 1 - eps*u3
                    if (s > 0.0f && s <= 1.0f) {
                        const double xd = (double)x, yd = (double)y;
                        const double d = __dsqrt_rn(__dadd_rn(__dmul_rn(xd, xd), __dmul_rn(yd, yd)));
                        const float u3 = u_hi(draw(key, i, a, 1));
                        const double rr = __dsub_rn(1.0, __dmul_rn(eps, (double)u3));
                        const double sc = __ddiv_rn(rr, d);
                        r.x = __double2float_rn(__dmul_rn(xd, sc));
                        r.y = __double2float_rn(__dmul_rn(yd, sc));
                        break;
                    }
                }
            }
        }
        out[j] = r;
    }
}

// 3D families (synth.generate3): 10 cube, 11 ball, 12 sphere
__global__ void gen3_kernel(int family, long long n, unsigned long long key, long long base, float lo,
                            float w, double eps, float* out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const unsigned long long i = (unsigned long long)(base + j);
        float r0 = 0.f, r1 = 0.f, r2 = 0.f;
        if (family == 10) {
            const unsigned long long z0 = draw(key, i, 0, 0), z1 = draw(key, i, 0, 1);
            r0 = __fadd_rn(__fmul_rn(u_hi(z0), w), lo);
            r1 = __fadd_rn(__fmul_rn(u_lo(z0), w), lo);
            r2 = __fadd_rn(__fmul_rn(u_hi(z1), w), lo);
        } else {
            for (int a = 0; a < kMaxAttempts; ++a) {
                const unsigned long long z0 = draw(key, i, a, 0), z1 = draw(key, i, a, 1);
                const float x = pm1(u_hi(z0)), y = pm1(u_lo(z0)), z = pm1(u_hi(z1));
                const float s = __fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)), __fmul_rn(z, z));
                if (family == 11) {
                    if (s <= 1.0f) {
                        r0 = x, r1 = y, r2 = z;
                        break;
                    }
                } else if (s > 0.0f && s <= 1.0f) {
                    const double xd = x, yd = y, zd = z;
                    const double d = __dsqrt_rn(
                        __dadd_rn(__dadd_rn(__dmul_rn(xd, xd), __dmul_rn(yd, yd)), __dmul_rn(zd, zd)));
                    const double rr = __dsub_rn(1.0, __dmul_rn(eps, (double)u_lo(z1)));
                    const double sc = __ddiv_rn(rr, d);
                    r0 = __double2float_rn(__dmul_rn(xd, sc));
                    r1 = __double2float_rn(__dmul_rn(yd, sc));
                    r2 = __double2float_rn(__dmul_rn(zd, sc));
                    break;
                }
            }
        }
        out[3 * j] = r0;
        out[3 * j + 1] = r1;
        out[3 * j + 2] = r2;
    }
}

}  // namespace

extern "C" int synth_generate(int family, long long n, unsigned long long seed, long long base,
                              double lo, double hi, double eps, void* d_out, void* stream) {
    const bool three = family >= 10 && family <= 12;
    if (!three && (family < 0 || family > 3)) return (int)cudaErrorInvalidValue;
    if (n < 0) return (int)cudaErrorInvalidValue;
    if (n == 0) return 0;
    unsigned long long key = mix64(seed * kGolden + kSalt);
    const float flo = (float)lo, fhi = (float)hi;
    const float w = fhi - flo;   // float32 RN subtraction, as numpy
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (n + 255) / 256;
    if (blocks > (long long)sms * 16) blocks = (long long)sms * 16;
    if (three)
        gen3_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(family, n, key, base, flo, w, eps,
                                                                        (float*)d_out);
    else
        gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(family, n, key, base, flo, w, eps,
                                                                       (float2*)d_out);
    return (int)cudaGetLastError();
}
