// Host-side helpers shared by the launchers (stree_host.cuh): cached TMA tensor-map encoding, SM count,
// once-per-device shared-memory attributes.  No device code.
#include <atomic>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "stree_host.cuh"

namespace stree {
namespace host {
namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

// the whole geometry of a map: a map is a pure function of it (the address is a UVA virtual address)
struct Key {
    uint64_t base, dims[4], strides[3];
    uint32_t box[4], dt, rank, swz, pad;
    bool operator==(const Key& o) const { return std::memcmp(this, &o, sizeof(Key)) == 0; }
};
struct KeyHash {
    size_t operator()(const Key& k) const {
        const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
        uint64_t h = 1469598103934665603ull;
        for (size_t i = 0; i < sizeof(Key) / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
        return (size_t)h;
    }
};

constexpr size_t kMaxCached = 16384;   // bounded: cleared when full (re-encoding is always correct)
std::mutex g_mu;
std::unordered_map<Key, CUtensorMap, KeyHash>& cache() {
    static auto* m = new std::unordered_map<Key, CUtensorMap, KeyHash>();
    return *m;
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, uint32_t rank, const void* base, const cuuint64_t* dims,
            const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    Key k;
    std::memset(&k, 0, sizeof(k));
    k.base = reinterpret_cast<uint64_t>(base);
    k.dt = (uint32_t)dt;
    k.rank = rank;
    k.swz = (uint32_t)swz;
    for (uint32_t i = 0; i < rank; ++i) {
        k.dims[i] = dims[i];
        k.box[i] = box[i];
        if (i + 1 < rank) k.strides[i] = strides[i];
    }
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = cache().find(k);
        if (it != cache().end()) {
            *m = it->second;
            return true;
        }
    }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (fn(m, dt, rank, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    std::lock_guard<std::mutex> lk(g_mu);
    if (cache().size() >= kMaxCached) cache().clear();
    cache().emplace(k, *m);
    return true;
}

}  // namespace

bool tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
             uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    return encode(m, dt, 2, base, dims, strides, box,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
}

bool tmap_4d_bf16(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b1,
                  uint32_t b2) {
    cuuint64_t dims[4] = {d0, d1, d2, d3};
    cuuint64_t strides[3] = {d0 * 2, d0 * d1 * 2, d0 * d1 * d2 * 2};
    cuuint32_t box[4] = {64, b1, b2, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box);
}

size_t tmap_cache_size() {
    std::lock_guard<std::mutex> lk(g_mu);
    return cache().size();
}

void tmap_cache_clear() {
    std::lock_guard<std::mutex> lk(g_mu);
    cache().clear();
}

int num_sms() {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    static std::atomic<int> cached[64];
    if (dev < 0 || dev >= 64) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }
    int c = cached[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev].store(v, std::memory_order_relaxed);
    return v;
}

cudaError_t smem_attr(const void* func, int bytes) {
    struct FKey {
        const void* f;
        int dev;
        bool operator==(const FKey& o) const { return f == o.f && dev == o.dev; }
    };
    struct FHash {
        size_t operator()(const FKey& k) const { return std::hash<const void*>()(k.f) ^ (size_t)k.dev * 0x9E3779B9u; }
    };
    static std::mutex mu;
    static auto* done = new std::unordered_map<FKey, int, FHash>();
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = done->find(FKey{func, dev});
        if (it != done->end() && it->second >= bytes) return cudaSuccess;
    }
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    int& v = (*done)[FKey{func, dev}];
    if (v < bytes) v = bytes;
    return cudaSuccess;
}

}  // namespace host
}  // namespace stree

// Debug / test hook (not part of the ABI): number of cached tensor maps; clear with clear != 0.
extern "C" long long stree_debug_tmap_cache(int clear) {
    if (clear) stree::host::tmap_cache_clear();
    return (long long)stree::host::tmap_cache_size();
}
