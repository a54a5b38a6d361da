// hbm_probe.cu — measurement tool (not product code): what a pure HBM read
// stream and variants of the segnorm inner loop achieve on this B200, to
// place td_segnorm against the real read ceiling rather than the copy peak.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_probe tools/hbm_probe.cu
//   tools/hbm_probe <GiB per operand>
//
// variants (each reads two equal buffers x, y once):
//   read_xor    : 16-B loads, integer xor reduce (memory ceiling, no math)
//   f2f_fp64    : bf16 -> f64 via F2F, d^2 and x^2 in fp64 (= td_segnorm nz=0)
//   int_fp64    : bf16 -> f64 via integer bit construction (no XU), fp64 math
//   bulk_fp64   : cp.async.bulk (TMA engine) 1-D copies into a 4-stage smem
//                 ring per CTA, mbarrier-synchronised, fp64 math from smem

#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <string>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldg_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

template <int U>
__global__ void __launch_bounds__(256, 4) read_xor(const uint4* x, const uint4* y, size_t n, unsigned* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256 * U) {
        uint4 a[U], b[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t j = i + (size_t)k * gridDim.x * 256;
            if (j < n) { a[k] = ldg_nc(x + j); b[k] = ldg_nc(y + j); } else { a[k] = make_uint4(0,0,0,0); b[k] = a[k]; }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) acc ^= a[k].x ^ a[k].y ^ a[k].z ^ a[k].w ^ b[k].x ^ b[k].y ^ b[k].z ^ b[k].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ double bf_f2f(uint32_t w, int hi) {
    return (double)__uint_as_float(hi ? (w & 0xffff0000u) : (w << 16));
}

// integer bit construction of the f64 high word; zero handled by select,
// subnormal/inf/nan flagged for a slow path (never taken with normal data)
__device__ __forceinline__ double bf_int(uint32_t w, int hi, bool& special) {
    const uint32_t b = hi ? (w >> 16) : (w & 0xffffu);
    const uint32_t m = b & 0x7fffu;
    const uint32_t e = m >> 7;
    special |= (e == 0xffu) | ((e == 0u) & (m != 0u));
    uint32_t t = m ? (m << 13) + 0x38000000u : 0u;
    t |= (b & 0x8000u) << 16;
    return __hiloint2double((int)t, 0);
}

template <int MODE, int U>
__global__ void __launch_bounds__(256, 4) seg_fp64(const uint4* x, const uint4* y, size_t n, double* out) {
    double d2 = 0, x2 = 0;
    bool special = false;
    for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256 * U) {
        uint4 a[U], b[U];
        bool ok[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            size_t j = i + (size_t)k * gridDim.x * 256;
            ok[k] = j < n;
            if (ok[k]) { a[k] = ldg_nc(x + j); b[k] = ldg_nc(y + j); }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            if (!ok[k]) continue;
            const uint32_t* aw = &a[k].x;
            const uint32_t* bw = &b[k].x;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                double xv, yv;
                if (MODE == 0) { xv = bf_f2f(aw[e >> 1], e & 1); yv = bf_f2f(bw[e >> 1], e & 1); }
                else if (MODE == 1) { xv = bf_int(aw[e >> 1], e & 1, special); yv = bf_int(bw[e >> 1], e & 1, special); }
                else { xv = bf_f2f(aw[e >> 1], e & 1); yv = bf_int(bw[e >> 1], e & 1, special); }
                const double d = xv - yv;
                d2 = fma(d, d, d2);
                x2 = fma(xv, xv, x2);
            }
        }
    }
    if (special) d2 += 1e300;
    if (d2 == 123.0 && x2 == 456.0) out[0] = d2;
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = d2 + x2;
}

// --- cp.async.bulk ring ------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(256, 1) bulk_fp64(const char* x, const char* y, size_t nbytes, double* out) {
    extern __shared__ __align__(128) char smem[];
    char* bx = smem;
    char* by = smem + STAGES * CHUNK;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * CHUNK);
    const size_t nchunks = nbytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_addr(&full[s])), "r"(2 * CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_addr(bx + s * CHUNK)), "l"(x + c * CHUNK), "r"(CHUNK), "r"(smem_addr(&full[s])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(smem_addr(by + s * CHUNK)), "l"(y + c * CHUNK), "r"(CHUNK), "r"(smem_addr(&full[s])) : "memory");
    };
    size_t c0 = blockIdx.x;
    int k = 0;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s) {
            size_t c = c0 + (size_t)s * gridDim.x;
            if (c < nchunks) issue(c, s);
        }
    double d2 = 0, x2 = 0;
    uint32_t phase = 0;
    for (size_t c = c0; c < nchunks; c += gridDim.x, ++k) {
        const int s = k % STAGES;
        // wait
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                     :: "r"(smem_addr(&full[s])), "r"(phase));
        const uint4* ax = reinterpret_cast<const uint4*>(bx + s * CHUNK);
        const uint4* ay = reinterpret_cast<const uint4*>(by + s * CHUNK);
        for (int v = threadIdx.x; v < CHUNK / 16; v += 256) {
            uint4 a = ax[v], b = ay[v];
            const uint32_t* aw = &a.x;
            const uint32_t* bw = &b.x;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const double xv = bf_f2f(aw[e >> 1], e & 1), yv = bf_f2f(bw[e >> 1], e & 1);
                const double d = xv - yv;
                d2 = fma(d, d, d2);
                x2 = fma(xv, xv, x2);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            size_t cn = c + (size_t)STAGES * gridDim.x;
            if (cn < nchunks) issue(cn, s);
        }
        if (s == STAGES - 1) phase ^= 1;
    }
    if (d2 == 123.0 && x2 == 456.0) out[0] = d2;
}

// "small": per-size read ceiling with L2 flushed (256 MiB memset) before each
// timed rep, one launch per rep between events — the regime of config 5's
// small tensors (td_segnorm there: 1 MiB 5.3 us, 16 MiB 11.5 us, 64 MiB
// 27.7 us per ncu).
static int small_sizes() {
    const size_t maxb = 256ull << 20;
    char *x, *y, *fl;
    unsigned* uout;
    CK(cudaMalloc(&x, maxb));
    CK(cudaMalloc(&y, maxb));
    CK(cudaMalloc(&fl, 256ull << 20));
    CK(cudaMalloc(&uout, 64));
    CK(cudaMemset(x, 1, maxb));
    CK(cudaMemset(y, 2, maxb));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t mib : {1, 4, 16, 64, 256}) {
        const size_t bytes = mib << 20, n16 = bytes / 16;
        auto time_it = [&](const char* name, auto launch) {
            std::vector<float> v;
            for (int r = 0; r < 23; ++r) {
                CK(cudaMemset(fl, r, 256ull << 20));
                cudaEventRecord(a);
                launch();
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) v.push_back(ms);
            }
            std::sort(v.begin(), v.end());
            const float med = v[v.size() / 2];
            printf("%4zu MiB x2  %-26s %8.2f us  %8.1f GB/s\n", mib, name, med * 1e3, 2.0 * bytes / (med / 1e3) / 1e9);
        };
        for (int per : {2, 4, 8}) {
            char nm[64];
            snprintf(nm, sizeof nm, "read_xor U=4 %d/SM", per);
            time_it(nm, [&] { read_xor<4><<<sms * per, 256>>>((const uint4*)x, (const uint4*)y, n16, uout); });
            snprintf(nm, sizeof nm, "read_xor U=8 %d/SM", per);
            time_it(nm, [&] { read_xor<8><<<sms * per, 256>>>((const uint4*)x, (const uint4*)y, n16, uout); });
        }
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "small") return small_sizes();
    double gib = argc > 1 ? atof(argv[1]) : 4.0;
    size_t bytes = (size_t)(gib * (1ull << 30));
    bytes &= ~((size_t)(1 << 20) - 1);
    char *x, *y;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMalloc(&y, bytes));
    // fill with bf16 ~N(0,1)-ish normal values (no zeros, no specials)
    std::vector<uint16_t> h(1 << 20);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(0x3f80 ^ (i * 2654435761u >> 20 & 0x7f)) | ((i & 1) << 15);
    for (size_t o = 0; o < bytes; o += h.size() * 2) {
        CK(cudaMemcpy(x + o, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(y + o, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    }
    double* out;
    unsigned* uout;
    CK(cudaMalloc(&out, 64));
    CK(cudaMalloc(&uout, 64));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t n16 = bytes / 16;
    auto time_it = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        const int reps = 10;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.1f GB/s  (%.3f ms per pass of %.2f GB)\n", name, 2.0 * bytes * reps / (ms / 1e3) / 1e9,
               ms / reps, 2.0 * bytes / 1e9);
    };
    time_it("read_xor U=4", [&] { read_xor<4><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, uout); });
    time_it("read_xor U=8", [&] { read_xor<8><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, uout); });
    time_it("f2f_fp64 U=4", [&] { seg_fp64<0, 4><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, out); });
    time_it("int_fp64 U=4", [&] { seg_fp64<1, 4><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, out); });
    time_it("mixed_fp64 U=4", [&] { seg_fp64<2, 4><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, out); });
    time_it("mixed_fp64 U=2", [&] { seg_fp64<2, 2><<<sms * 4, 256>>>((const uint4*)x, (const uint4*)y, n16, out); });
    {
        constexpr int ST = 4, CH = 16384;
        const int sm_bytes = 2 * ST * CH + 64;
        CK(cudaFuncSetAttribute(bulk_fp64<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
        time_it("bulk_fp64 4x16K x2", [&] { bulk_fp64<ST, CH><<<sms, 256, sm_bytes>>>(x, y, bytes, out); });
    }
    {
        constexpr int ST = 6, CH = 8192;
        const int sm_bytes = 2 * ST * CH + 64;
        CK(cudaFuncSetAttribute(bulk_fp64<ST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
        time_it("bulk_fp64 6x8K x2 (2/SM)", [&] { bulk_fp64<ST, CH><<<sms * 2, 256, sm_bytes>>>(x, y, bytes, out); });
    }
    CK(cudaGetLastError());
    return 0;
}
