// Host side of the TMA helpers: cuTensorMapEncodeTiled through the runtime's
// driver entry point, with a small cache keyed by (pointer, dims, box).
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "tma.cuh"

namespace vpfv {

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool tma_available() { return encode_fn() != nullptr; }

namespace {
struct Key {
    const void *ptr;
    int rank;
    unsigned long long dims[4];
    unsigned box[4];
    bool operator==(const Key &o) const {
        if (ptr != o.ptr || rank != o.rank) return false;
        for (int i = 0; i < 4; ++i)
            if (dims[i] != o.dims[i] || box[i] != o.box[i]) return false;
        return true;
    }
};
struct KeyHash {
    size_t operator()(const Key &k) const {
        size_t h = reinterpret_cast<size_t>(k.ptr) ^ (size_t)k.rank;
        for (int i = 0; i < 4; ++i) h = h * 1000003u ^ (size_t)(k.dims[i] * 131 + k.box[i]);
        return h;
    }
};
}  // namespace

bool tma_map(const void *ptr, int rank, const unsigned long long *dims, const unsigned long long *strides,
             const unsigned *box, CUtensorMap *out) {
    static std::mutex mu;
    static std::unordered_map<Key, CUtensorMap, KeyHash> cache;
    Key key{ptr, rank, {0, 0, 0, 0}, {0, 0, 0, 0}};
    for (int i = 0; i < rank; ++i) {
        key.dims[i] = dims[i];
        key.box[i] = box[i];
    }
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t d[4], st[3];
    cuuint32_t b[4], es[4] = {1, 1, 1, 1};
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
    }
    for (int i = 0; i < rank - 1; ++i) st[i] = strides[i];
    static int promo = -1;  // L2 promotion of TMA fetches (VPFV_TMA_PROMO = 0/64/128/256)
    if (promo < 0) {
        const char *e = getenv("VPFV_TMA_PROMO");
        promo = e ? atoi(e) : 256;
    }
    const CUtensorMapL2promotion pr = promo == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                      : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                      : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                     : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    CUtensorMap m;
    if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void *>(ptr), d, st, b, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
        return false;
    if (cache.size() > 512) cache.clear();
    cache.emplace(key, m);
    *out = m;
    return true;
}

}  // namespace vpfv
