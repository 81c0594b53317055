// cascade.cu — the C ABI of include/cascade.h: model weights, sessions,
// the verification-step graph and greedy acceptance.
//
// One verification step of width T = K+1:
//   H2D step params -> embed+norm
//   per layer: QKV GEMV -> attention (RoPE, KV append, split-KV) -> combine
//              -> O GEMV (+residual) -> route (norm, router, top-k, union)
//              -> expert gate/up GEMV (SiLU fused) -> expert down GEMV
//              -> [EP all-reduce] -> combine (+residual, next norm)
//   LM head GEMV (+argmax) -> accept (greedy prefix, KV commit, utility)
//   -> D2H result
// captured once per T into a CUDA graph; routing, context length and the
// pending token live in device memory so the graph is replayed unchanged.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "attention.cuh"
#include "cascade.h"
#include "common.cuh"
#include "ffn_ring.cuh"
#include "gemv.cuh"
#include "init.cuh"
#include "moe.cuh"

#ifndef CASCADE_GIT
#define CASCADE_GIT "unknown"
#endif

using namespace cascade;

// ---------------------------------------------------------------- errors
static thread_local std::string g_err;

static int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_err(CASCADE_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

extern "C" size_t cascade_last_error(char* buf, size_t n) {
    if (buf && n) {
        const size_t c = std::min(n - 1, g_err.size());
        std::memcpy(buf, g_err.data(), c);
        buf[c] = 0;
    }
    return g_err.size();
}

// internal (hidden): lets decode.cpp report through the same error slot
extern "C" int cascade_internal_set_error(int code, const char* msg) { return set_err(code, msg ? msg : ""); }

extern "C" const char* cascade_build_info(void) { return "sm_100a " CASCADE_GIT; }

// ---------------------------------------------------------------- NCCL (dlopen)
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
struct NcclApi {
    void* h = nullptr;
    int (*GetUniqueId)(nccl_uid_t*) = nullptr;
    int (*CommInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*CommDestroy)(nccl_comm_t) = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
static NcclApi g_nccl;
static int nccl_load() {
    if (g_nccl.h) return CASCADE_OK;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return set_err(CASCADE_ERUNTIME, std::string("dlopen libnccl: ") + dlerror());
    g_nccl.GetUniqueId = (int (*)(nccl_uid_t*))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (int (*)(nccl_comm_t*, int, nccl_uid_t, int))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t))dlsym(
        h, "ncclAllReduce");
    g_nccl.CommDestroy = (int (*)(nccl_comm_t))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
    if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy)
        return set_err(CASCADE_ERUNTIME, "libnccl is missing symbols");
    g_nccl.h = h;
    return CASCADE_OK;
}
constexpr int kNcclFloat32 = 7;
constexpr int kNcclSum = 0;

extern "C" int cascade_ep_unique_id(void* out, size_t n) {
    if (!out || n < sizeof(nccl_uid_t)) return set_err(CASCADE_EINVAL, "unique id buffer < 128 bytes");
    int rc = nccl_load();
    if (rc) return rc;
    nccl_uid_t id;
    if (g_nccl.GetUniqueId(&id) != 0) return set_err(CASCADE_ERUNTIME, "ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof(id));
    return CASCADE_OK;
}

// ---------------------------------------------------------------- geometry
static int validate(const cascade_geometry* g) {
    if (!g) return set_err(CASCADE_EINVAL, "geometry is NULL");
    auto bad = [](const std::string& m) { return set_err(CASCADE_EINVAL, "cascade_geometry: " + m); };
    // the reference's own ExpertConfig rules (expert_model.hpp:37-50)
    if (g->num_layers < 1) return bad("num_layers must be >= 1");
    if (g->top_k < 1 || g->shared_experts < 0 || g->top_k > g->experts_per_layer)
        return bad("need 1 <= top_k <= experts_per_layer and shared_experts >= 0");
    // limits of this implementation
    if (g->num_layers > CASCADE_MAX_LAYERS) return bad("num_layers > 128");
    if (g->experts_per_layer > kMaxExperts) return bad("experts_per_layer > 128 (expert_model.hpp:96)");
    if (g->top_k > kMaxTopK) return bad("top_k > 16");
    if (g->shared_experts > 16) return bad("shared_experts > 16");
    if (g->d_model < 256 || g->d_model % 256 || g->d_model > 8192) return bad("d_model must be a multiple of 256 in [256, 8192]");
    if (g->d_ff < 32 || g->d_ff % 32) return bad("d_ff must be a positive multiple of 32");
    if (g->head_dim != 32 && g->head_dim != 64 && g->head_dim != 128) return bad("head_dim must be 32, 64 or 128");
    if (g->n_kv_heads < 1 || g->n_heads < 1 || g->n_heads % g->n_kv_heads) return bad("n_heads must be a multiple of n_kv_heads");
    if ((g->n_heads / g->n_kv_heads) * kMaxT > kAttnMaxRows) return bad("n_heads / n_kv_heads must be <= 8");
    if ((g->n_heads * g->head_dim) % 64) return bad("n_heads*head_dim must be a multiple of 64");
    if (((g->n_heads + 2 * g->n_kv_heads) * g->head_dim) % 64) return bad("(H+2KV)*head_dim must be a multiple of 64");
    if (g->vocab < 128 || g->vocab % 128) return bad("vocab must be a positive multiple of 128");
    if (((g->n_heads + 2 * g->n_kv_heads) * g->head_dim) % 128) return bad("(H+2KV)*head_dim must be a multiple of 128");
    if (!(g->rope_theta > 0.f)) return bad("rope_theta must be > 0");
    if (!(g->norm_eps > 0.f)) return bad("norm_eps must be > 0");
    if (!(g->router_scale > 0.f)) return bad("router_scale must be > 0");
    return CASCADE_OK;
}

extern "C" int cascade_geometry_validate(const cascade_geometry* g) { return validate(g); }

struct Dims {
    int L, E, k, S, d, f, H, KV, hd, V, qkvd, hq;
    long long w13_vec, w2_vec, wqkv_vec, wo_vec, lm_vec;  // uint4 counts
    explicit Dims(const cascade_geometry& g) {
        L = g.num_layers; E = g.experts_per_layer; k = g.top_k; S = g.shared_experts;
        d = g.d_model; f = g.d_ff; H = g.n_heads; KV = g.n_kv_heads; hd = g.head_dim; V = g.vocab;
        hq = H * hd;
        qkvd = (H + 2 * KV) * hd;
        w13_vec = (long long)2 * f * d / 8;
        w2_vec = (long long)d * f / 8;
        wqkv_vec = (long long)qkvd * d / 8;
        wo_vec = (long long)d * hq / 8;
        lm_vec = (long long)V * d / 8;
    }
};

static int g_route_stage = 1;  // CASCADE_ROUTE_STAGE=0: read router rows from global (A/B: staging measured faster)
static bool route_staged(const Dims& D, int shared_gate) {
    return g_route_stage && (size_t)(D.E + (shared_gate ? 1 : 0)) * D.d * 2 <= (size_t)kRouteStageBytes;
}
static int g_route_cluster = 1;  // CASCADE_ROUTE_CLUSTER=0: large routers read from global by one CTA
// CTAs per token: routers larger than one CTA's staging budget are split
// over a cluster so every row is staged in shared memory before the wait.
static int route_cluster(const Dims& D, int shared_gate) {
    const size_t bytes = (size_t)(D.E + (shared_gate ? 1 : 0)) * D.d * 2;
    if (route_staged(D, shared_gate) || !g_route_cluster || !g_route_stage) return 1;
    const int C = (int)((bytes + kRouteStageBytes - 1) / kRouteStageBytes);
    return C <= 8 ? C : 1;
}
static size_t route_smem_bytes(const Dims& D, int shared_gate) {
    const int rows = D.E + (shared_gate ? 1 : 0);
    const int C = route_cluster(D, shared_gate);
    if (C > 1) return (size_t)D.d * 4 + (size_t)((rows + C - 1) / C) * D.d * 2;
    return (size_t)D.d * 4 + (route_staged(D, shared_gate) ? (size_t)rows * D.d * 2 : 0);
}

static void local_experts(int E, int rank, int size, int& lo, int& hi) {
    lo = (int)((long long)E * rank / size);
    hi = (int)((long long)E * (rank + 1) / size);
}
static int local_shared(int S, int rank, int size) {
    int n = 0;
    for (int b = 0; b < S; ++b) n += (b % size) == rank;
    return n;
}

extern "C" int cascade_model_bytes(const cascade_geometry* g, int ep_rank, int ep_size, uint64_t* out) {
    int rc = validate(g);
    if (rc) return rc;
    if (!out || ep_size < 1 || ep_rank < 0 || ep_rank >= ep_size) return set_err(CASCADE_EINVAL, "bad EP rank/size");
    Dims D(*g);
    int lo, hi;
    local_experts(D.E, ep_rank, ep_size, lo, hi);
    const long long nb = (hi - lo) + local_shared(D.S, ep_rank, ep_size);
    uint64_t per_layer = (uint64_t)(D.wqkv_vec + D.wo_vec + nb * (D.w13_vec + D.w2_vec)) * 16 +
                         (uint64_t)2 * D.d * 2 + (uint64_t)(D.E + 1) * D.d * 2;
    *out = per_layer * D.L + (uint64_t)D.V * D.d * 2 * 2 + (uint64_t)D.d * 2;
    return CASCADE_OK;
}

// ---------------------------------------------------------------- model
struct LayerW {
    uint16_t* attn_norm = nullptr;
    uint16_t* ffn_norm = nullptr;
    uint16_t* router = nullptr;  // [E + 1][d] (row E = shared gate when present)
    uint4* wqkv = nullptr;
    uint4* wo = nullptr;
    uint4* w13 = nullptr;        // [n_blocks][2f x d]
    uint4* w2 = nullptr;         // [n_blocks][d x f]
};

struct cascade_model {
    cascade_geometry g{};
    uint64_t seed = 0;
    int device = 0;
    int num_sms = 148;
    int ep_rank = 0, ep_size = 1;
    int e_lo = 0, e_hi = 0, n_shared_local = 0, n_blocks = 0;
    std::vector<LayerW> layers;
    uint16_t* embed = nullptr;
    uint16_t* final_norm = nullptr;
    uint4* lm_head = nullptr;
    std::vector<void*> allocs;
    uint64_t bytes = 0;
    nccl_comm_t comm = nullptr;
    // dense matrices on the tcgen05 engine (gemv_umma.cuh, UMMA layout) vs the
    // mma.sync engine (gemv.cuh, A-frag layout), per matrix: bit 0 QKV, bit 1
    // O projection, bit 2 LM head.  Default all three; in-graph A/B of the
    // masks (profiles/r01/ab) puts them within noise of each other on the
    // K=0..8 mean, tcgen05 ahead on QKV.  CASCADE_DENSE_UMMA=<mask> overrides.
    int umma_mask = 7;
    bool umma_qkv() const { return umma_mask & 1; }
    bool umma_o() const { return umma_mask & 2; }
    bool umma_lm() const { return umma_mask & 4; }
};

template <typename T>
static int dalloc(cascade_model* m, T** p, size_t bytes) {
    void* v = nullptr;
    CK(cudaMalloc(&v, bytes));
    m->allocs.push_back(v);
    m->bytes += bytes;
    *p = (T*)v;
    return CASCADE_OK;
}

static uint64_t key_of(const cascade_model* m, int kind, int layer, int expert) {
    return cascade_tensor_key(m->seed, cascade_tensor_id(kind, layer, expert));
}

static int init_afrag(cascade_model* m, uint4* dst, int rows, int cols, int rowmap, int k0, int k1, int k2,
                      int layer, int expert, int n0 = 0, int n1 = 0, int umma = 0) {
    InitParams p{};
    p.umma = umma;
    p.dst = dst;
    p.n_vec = (long long)rows * cols / 8;
    p.n_ks = cols / 16;
    p.rowmap = rowmap;
    p.n0 = n0;
    p.n1 = n1;
    p.cols = cols;
    const int kinds[3] = {k0, k1, k2};
    for (int i = 0; i < 3; ++i) {
        const int kd = kinds[i] ? kinds[i] : k0;
        p.key[i] = key_of(m, kd, layer, expert);
        p.scale[i] = cascade_kind_scale(kd, cols, m->g.router_scale);
    }
    const int blocks = (int)std::min<long long>((p.n_vec + 255) / 256, (long long)m->num_sms * 16);
    init_afrag_kernel<<<blocks, 256>>>(p);
    CK(cudaGetLastError());
    return CASCADE_OK;
}

static int init_plain(cascade_model* m, uint16_t* dst, int rows, int cols, int kind, int layer, int expert,
                      int fan_in) {
    const long long n = (long long)rows * cols;
    const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)m->num_sms * 16);
    init_plain_kernel<<<blocks, 256>>>(dst, n, cols, n, key_of(m, kind, layer, expert),
                                       cascade_kind_scale(kind, fan_in, m->g.router_scale), 0);
    CK(cudaGetLastError());
    return CASCADE_OK;
}

extern "C" int cascade_model_destroy(cascade_model* m) {
    if (!m) return CASCADE_OK;
    cudaSetDevice(m->device);
    cudaDeviceSynchronize();
    for (void* p : m->allocs) cudaFree(p);
    if (m->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(m->comm);
    delete m;
    return CASCADE_OK;
}

static int model_create(const cascade_geometry* g, uint64_t seed, int device, int ep_rank, int ep_size,
                        const void* uid, cascade_model** out) {
    int rc = validate(g);
    if (rc) return rc;
    if (!out) return set_err(CASCADE_EINVAL, "out is NULL");
    if (ep_size < 1 || ep_rank < 0 || ep_rank >= ep_size) return set_err(CASCADE_EINVAL, "bad EP rank/size");
    if (ep_size > g->experts_per_layer) return set_err(CASCADE_EINVAL, "ep_size > experts_per_layer");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(CASCADE_EINVAL, "device index out of range");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return set_err(CASCADE_ERUNTIME, "this library is built for sm_100a (B200)");

    cascade_model* m = new cascade_model();
    m->g = *g;
    m->seed = seed;
    m->device = device;
    m->num_sms = prop.multiProcessorCount;
    m->ep_rank = ep_rank;
    m->ep_size = ep_size;
    local_experts(g->experts_per_layer, ep_rank, ep_size, m->e_lo, m->e_hi);
    m->n_shared_local = local_shared(g->shared_experts, ep_rank, ep_size);
    m->n_blocks = (m->e_hi - m->e_lo) + m->n_shared_local;
    if (const char* v = getenv("CASCADE_DENSE_UMMA")) m->umma_mask = atoi(v) & 7;
    Dims D(*g);
    m->layers.resize(D.L);

    auto fail = [&](int code) {
        std::string msg = g_err;
        cascade_model_destroy(m);
        g_err = msg;
        return code;
    };

    for (int l = 0; l < D.L; ++l) {
        LayerW& w = m->layers[l];
        if ((rc = dalloc(m, &w.attn_norm, D.d * 2)) || (rc = dalloc(m, &w.ffn_norm, D.d * 2)) ||
            (rc = dalloc(m, &w.router, (size_t)(D.E + 1) * D.d * 2)) ||
            (rc = dalloc(m, &w.wqkv, D.wqkv_vec * 16)) || (rc = dalloc(m, &w.wo, D.wo_vec * 16)) ||
            (rc = dalloc(m, &w.w13, (size_t)m->n_blocks * D.w13_vec * 16)) ||
            (rc = dalloc(m, &w.w2, (size_t)m->n_blocks * D.w2_vec * 16)))
            return fail(rc);
        if ((rc = init_plain(m, w.attn_norm, 1, D.d, CASCADE_T_ATTN_NORM, l, 0, D.d)) ||
            (rc = init_plain(m, w.ffn_norm, 1, D.d, CASCADE_T_FFN_NORM, l, 0, D.d)) ||
            (rc = init_plain(m, w.router, D.E, D.d, CASCADE_T_ROUTER, l, 0, D.d)))
            return fail(rc);
        if (g->shared_gate) {
            if ((rc = init_plain(m, w.router + (size_t)D.E * D.d, 1, D.d, CASCADE_T_SHARED_GATE, l, 0, D.d)))
                return fail(rc);
        } else {
            CK(cudaMemset(w.router + (size_t)D.E * D.d, 0, D.d * 2));
        }
        if ((rc = init_afrag(m, w.wqkv, D.qkvd, D.d, ROWMAP_QKV, CASCADE_T_WQ, CASCADE_T_WK, CASCADE_T_WV, l, 0,
                             D.hq, D.KV * D.hd, m->umma_qkv())) ||
            (rc = init_afrag(m, w.wo, D.d, D.hq, ROWMAP_SIMPLE, CASCADE_T_WO, 0, 0, l, 0, 0, 0, m->umma_o())))
            return fail(rc);
        for (int b = 0; b < m->n_blocks; ++b) {
            // global expert index: local routed experts, then local shared blocks
            int ge;
            if (b < m->e_hi - m->e_lo) {
                ge = m->e_lo + b;
            } else {
                int lb = b - (m->e_hi - m->e_lo), seen = 0;
                ge = -1;
                for (int s = 0; s < D.S; ++s)
                    if (s % ep_size == ep_rank) {
                        if (seen == lb) { ge = D.E + s; break; }
                        ++seen;
                    }
            }
            if ((rc = init_afrag(m, w.w13 + (size_t)b * D.w13_vec, 2 * D.f, D.d, ROWMAP_GATEUP, CASCADE_T_W_GATE,
                                 CASCADE_T_W_UP, 0, l, ge)) ||
                (rc = init_afrag(m, w.w2 + (size_t)b * D.w2_vec, D.d, D.f, ROWMAP_SIMPLE, CASCADE_T_W_DOWN, 0, 0,
                                 l, ge)))
                return fail(rc);
        }
    }
    if ((rc = dalloc(m, &m->embed, (size_t)D.V * D.d * 2)) || (rc = dalloc(m, &m->final_norm, D.d * 2)) ||
        (rc = dalloc(m, &m->lm_head, D.lm_vec * 16)))
        return fail(rc);
    if ((rc = init_plain(m, m->embed, D.V, D.d, CASCADE_T_EMBED, 0, 0, D.d)) ||
        (rc = init_plain(m, m->final_norm, 1, D.d, CASCADE_T_FINAL_NORM, 0, 0, D.d)) ||
        (rc = init_afrag(m, m->lm_head, D.V, D.d, ROWMAP_SIMPLE, CASCADE_T_LM_HEAD, 0, 0, 0, 0, 0, 0, m->umma_lm())))
        return fail(rc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        set_err(CASCADE_ECUDA, std::string("weight init: ") + cudaGetErrorString(e));
        return fail(CASCADE_ECUDA);
    }
    // CASCADE_EP_NOCOMM=1 (tests only): an expert shard without a communicator,
    // so one GPU can run every shard of a world and check the partition
    const char* nocomm = getenv("CASCADE_EP_NOCOMM");
    if ((ep_size > 1 || uid) && !(nocomm && nocomm[0] == '1')) {  // an expert-parallel model (any world size, 1 included) owns a communicator
        if ((rc = nccl_load())) return fail(rc);
        if (!uid) {
            set_err(CASCADE_EINVAL, "nccl_unique_id is NULL for ep_size > 1");
            return fail(CASCADE_EINVAL);
        }
        nccl_uid_t id;
        std::memcpy(&id, uid, sizeof(id));
        const int nr = g_nccl.CommInitRank(&m->comm, ep_size, id, ep_rank);
        if (nr != 0) {
            set_err(CASCADE_ERUNTIME, std::string("ncclCommInitRank: ") +
                                          (g_nccl.GetErrorString ? g_nccl.GetErrorString(nr) : "error"));
            m->comm = nullptr;
            return fail(CASCADE_ERUNTIME);
        }
    }
    *out = m;
    return CASCADE_OK;
}

extern "C" int cascade_model_create(const cascade_geometry* g, uint64_t seed, int device, cascade_model** out) {
    return model_create(g, seed, device, 0, 1, nullptr, out);
}

extern "C" int cascade_model_create_ep(const cascade_geometry* g, uint64_t seed, int device, int ep_rank,
                                       int ep_size, const void* uid, cascade_model** out) {
    return model_create(g, seed, device, ep_rank, ep_size, uid, out);
}

// ---------------------------------------------------------------- accept
struct AcceptParams {
    const StepParams* sp;
    DevState* st;
    unsigned long long* keys;
    const int* tokens_used;
    const unsigned long long* stamps;  // [0] start, [1+2l] attn l, [2+2l] moe l, [1+2L] lm head
    const int* union_size;
    cascade_verify_out* res;
    int T, L, S;
    unsigned long long* trace;  // start slot; slot+1 receives the step end
};

__global__ void accept_kernel(AcceptParams p) {
    griddep_wait();
    CTA_TRACE(p.trace);
    if (threadIdx.x != 0) return;
    const uint64_t t_end = globaltimer();
    if (p.trace) p.trace[1] = t_end;
    cascade_verify_out r;
    memset(&r, 0, sizeof(r));
    int am[kMaxT];
    for (int t = 0; t < p.T; ++t) {
        am[t] = argmax_key_index(p.keys[t]);
        p.keys[t] = 0ull;
        r.argmax[t] = am[t];
    }
    const StepParams sp = *p.sp;
    int acc = 0;
    if (sp.mode == 0) {
        while (acc < p.T - 1 && am[acc] == p.tokens_used[acc + 1]) ++acc;
        for (int i = 0; i < acc; ++i) r.tokens[i] = p.tokens_used[i + 1];
        r.tokens[acc] = am[acc];
        r.accepted = acc;
        r.emitted = acc + 1;
        if (sp.commit) {
            p.st->cache_len += acc + 1;
            p.st->pending = am[acc];
        }
    } else {
        r.accepted = 0;
        r.emitted = 0;
        if (sp.commit) p.st->cache_len += p.T;
    }
    p.st->steps += 1;
    r.n_tokens = p.T;
    r.cache_len = p.st->cache_len;
    const double t0 = (double)p.stamps[0];
    double att = (double)p.stamps[1] - t0, exp_t = 0.0;
    double active = 0.0;
    for (int l = 0; l < p.L; ++l) {
        const double a = (double)p.stamps[1 + 2 * l];
        const double mo = (double)p.stamps[2 + 2 * l];
        const double nx = (double)p.stamps[1 + 2 * (l + 1)];  // next attn start or LM head start
        att += mo - a;
        exp_t += nx - mo;
        active += (double)(p.union_size[l] + p.S);
    }
    r.attention_time = att;
    r.expert_time = exp_t;
    r.sampling_time = (double)t_end - (double)p.stamps[1 + 2 * p.L];
    r.draft_time = sp.draft_ns;
    r.total = r.attention_time + r.expert_time + r.draft_time + r.sampling_time;
    r.active_experts_per_layer = active / p.L;
    r.verify_ns = (double)t_end - t0;
    r.utility = (sp.t_base_ns > 0.0 && r.emitted > 0) ? (double)r.emitted * sp.t_base_ns / r.total : 0.0;
    *p.res = r;
}

// One shared-memory carveout for every kernel of the step: an SM that ran a
// large-smem kernel otherwise stays configured for it (tiny L1) until
// it drains, and the L1-cached activation reads of the next GEMV suffer.
static int g_carveout = 58;  // percent of 228 KB -> the 132 KB configuration
template <typename K>
static cudaError_t carve(K k) {
    return g_carveout > 0 ? cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout)
                          : cudaSuccess;
}
template <int NT>
static cudaError_t carve_gemv() {
    cudaError_t e = carve(stream_gemv_kernel<NT, EPI_STORE>);
    if (e == cudaSuccess) e = carve(stream_gemv_kernel<NT, EPI_ADD>);
    if (e == cudaSuccess) e = carve(stream_gemv_kernel<NT, EPI_GATEUP>);
    if (e == cudaSuccess) e = carve(stream_gemv_kernel<NT, EPI_DOWN>);
    if (e == cudaSuccess) e = carve(stream_gemv_kernel<NT, EPI_ARGMAX>);
    return e;
}
static cudaError_t set_carveouts(int hd) {
    if (const char* v = getenv("CASCADE_CARVEOUT")) g_carveout = atoi(v);
    cudaError_t e = carve_gemv<1>();
    if (e == cudaSuccess) e = carve_gemv<2>();
    if (e == cudaSuccess) e = carve(stream_gemv_umma_kernel<UEPI_STORE>);
    if (e == cudaSuccess) e = carve(stream_gemv_umma_kernel<UEPI_ADD>);
    if (e == cudaSuccess) e = carve(stream_gemv_umma_kernel<UEPI_ARGMAX>);
    if (e == cudaSuccess) e = carve(moe_route_kernel);
    if (e == cudaSuccess) e = carve(moe_combine_kernel);
    if (e == cudaSuccess) e = carve(embed_norm_kernel);
    if (e == cudaSuccess) e = carve(attn_combine_kernel);
    if (e == cudaSuccess) e = carve(accept_kernel);
    if (e == cudaSuccess) e = hd == 32 ? carve(attn_partial_kernel<32>) : hd == 64 ? carve(attn_partial_kernel<64>) : carve(attn_partial_kernel<128>);
    return e;
}

template <int NT>
static cudaError_t gemv_smem_attr() {
    const int sm = gemv_smem_bytes<NT>();
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_kernel<NT, EPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_kernel<NT, EPI_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_kernel<NT, EPI_GATEUP>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_kernel<NT, EPI_DOWN>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_kernel<NT, EPI_ARGMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    return e;
}

// ---------------------------------------------------------------- SM rate calibration
// Streaming rates differ by SM by a few percent, consistently (profiles:
// scripts/sm_speed.py), and a static equal split waits for the slowest
// SM.  At session creation every CTA of a 2-per-SM grid streams an equal
// slice of the expert weights with the GEMV's load pattern; the per-SM
// rates give the piece weights of the expert GEMVs' grid-wide split.
__global__ void __launch_bounds__(kGemvThreads, 2) sm_rate_probe_kernel(const uint4* src, long long per_cta_vec,
                                                                       unsigned long long* out) {
    const uint64_t pol = policy_evict_first();
    const uint4* base = src + (long long)blockIdx.x * per_cta_vec;
    __syncthreads();
    const unsigned long long t0 = globaltimer_raw();
    uint32_t acc = 0;
    for (long long i = threadIdx.x; i < per_cta_vec; i += (long long)blockDim.x * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long j = i + (long long)u * blockDim.x;
            v[u] = j < per_cta_vec ? ldg_stream(base + j, pol) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    __syncthreads();
    const unsigned long long t1 = globaltimer_raw();
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        out[blockIdx.x * 2] = smid | ((unsigned long long)(acc & 1u) << 40);  // acc keeps the loads alive
        out[blockIdx.x * 2 + 1] = t1 - t0;
    }
}

// Cluster size for the split-K dense GEMV over n_units 128-row units: the
// largest C <= 8 with n_units * C <= SMs whose clusters can all be resident
// at once (one wave); 0 = use the stream-K path.
static int pick_cluster(const cascade_model* m, int n_units, int smem_bytes) {
    for (int C = std::min(kCMaxC, m->num_sms / std::max(n_units, 1)); C >= 2; --C) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n_units * C);
        cfg.blockDim = dim3(kUThreads);
        cfg.dynamicSmemBytes = smem_bytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, dense_gemv_cluster_kernel<UEPI_STORE>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (getenv("CASCADE_DEBUG_CLUSTER")) fprintf(stderr, "cluster C=%d: %d clusters active (need %d)\n", C, n, n_units);
        if (n >= n_units) return C;
    }
    return 0;
}

static cudaError_t launch_dense_cluster(int epi, const UGemvParams& p, int C, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.n_st * C);
    cfg.blockDim = dim3(kUThreads);
    cfg.dynamicSmemBytes = dense_cluster_smem_bytes(p.ring_stages, p.stage_ks);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = C;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (epi == UEPI_ADD) return cudaLaunchKernelEx(&cfg, dense_gemv_cluster_kernel<UEPI_ADD>, p);
    return cudaLaunchKernelEx(&cfg, dense_gemv_cluster_kernel<UEPI_STORE>, p);
}

// ---------------------------------------------------------------- session
struct Taps {
    uint16_t* xn_moe = nullptr;   // [L][16][d]
    float* logits = nullptr;      // [L][16][E+1]
    int* topk_id = nullptr;       // [L][16][k]
    float* topk_w = nullptr;      // [L][16][k]
    float* moe_out = nullptr;     // [L][16][d]
    float* final_logits = nullptr;// [16][V]
    uint16_t* xn_attn = nullptr;  // [L][16][d]
    float* x_mid = nullptr;       // [L][16][d] residual after attention
    float* x_in = nullptr;        // [L][16][d] residual entering the layer
};

struct cascade_session {
    cascade_model* m = nullptr;
    int max_ctx = 0, k_max = 0, max_chunks = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::vector<void*> allocs;
    StepParams* d_params = nullptr;
    // Pinned step parameters, one slot per width T: the step graph of width
    // T copies slot T when it executes, so a slot is only rewritten after
    // the stream drained (set_params) and enqueued graphs of other widths
    // never see another call's parameters.
    StepParams* h_params = nullptr;
    int32_t drafts[kMaxT] = {};  // token slots the next enqueue-only step verifies (last prefill chunk / verify)
    int len_hi = 0;              // upper bound of the device KV length (exact after every host sync point)
    int user_ctx = 0;            // max_ctx as created: committed KV length never exceeds it
    DevState* d_state = nullptr;
    cascade_verify_out* d_result = nullptr;
    cascade_verify_out* h_result = nullptr;
    float* x = nullptr;
    uint16_t* xn = nullptr;      // MoE input (B-frag, expert GEMVs)
    uint16_t* xn_u = nullptr;    // attention / final-norm output (UMMA B layout for tcgen05 QKV / LM head)
    float* upartial = nullptr;   // tcgen05 engine split-unit partials
    int* ucounters = nullptr;
    float* qkv = nullptr;
    float* attn_part = nullptr;
    uint16_t* attn_out = nullptr;
    float* logits_router = nullptr;
    int* topk_id = nullptr;
    float* topk_w = nullptr;
    float* gsh = nullptr;
    int* list = nullptr;
    int* count = nullptr;
    int* route_rank = nullptr;
    int* union_size = nullptr;
    uint16_t* hbuf = nullptr;
    float* ycontrib = nullptr;
    float4* partial = nullptr;
    int* counters = nullptr;
    unsigned long long* keys = nullptr;
    unsigned long long* stamps = nullptr;
    int* tokens_used = nullptr;
    float2* rope = nullptr;
    unsigned long long* trace = nullptr;  // per-kernel start stamps of the last step
    int trace_kind[kMaxT + 1][2048] = {};
    int trace_n[kMaxT + 1] = {};
    bool prefetch = true;
    int l2_prologue = 0;  // measured slower (down-proj ranges exceed L2; QKV prefetch slows the combine)
    int gemv_trigger = 1;  // early launch_dependents: the down GEMV builds its union and requests its first weights while gate/up drains
    int down_early = 1;
    int umma_prologue = 1;
    int attn_fused = 0;    // chunk combine inside the attention kernel (last item per KV head); A/B: the separate combine is as fast or faster
    int ffn_trigger = 0;   // fused FFN: launch_dependents right after the wait (A/B: off is faster)
    int ffn_fused = 1;     // expert gate/up + down in one launch (expert_ffn_kernel; CASCADE_FFN_FUSED=0: two launches)
    int unit_pieces = 1;   // expert GEMVs: whole super-tile per CTA when they nearly fill the grid (CASCADE_UNIT_PIECES=0: always stream-K)
    int ffn_ring = 1;      // fused FFN with one TMA stream per SM for T <= 8 (ffn_ring.cuh; CASCADE_FFN_RING=0: register engine)
    // attention chunk tiles (CASCADE_ATTN_KSPLIT): 0 one warp per 16-row tile,
    // 1 key split, 2 transposed key split, 3 per step width the one with
    // fewer mma per warp (all four give bitwise-identical partials)
    int attn_ksplit = 3;
    int ring_max_t = 8;    // ring engine up to this many tokens (CASCADE_RING_MAXT; 16: every width)
    int ring_slot_major = 0;  // ring engine: per-slot pieces for large experts (CASCADE_RING_SLOTMAJOR=1)
    int ring_dn_l2 = 0;    // ring engine: down stages L2-prefetched at the gate/up -> down transition (CASCADE_RING_DNPF)
    int ring_unit_pieces = 0;  // ring engine: allow one-super-tile pieces (CASCADE_RING_UNIT=1)
    int ffn_fma = 0;       // fused FFN at T = 1 on CUDA-core FMAs instead of mma.sync (CASCADE_FFN_FMA=1; A/B: profiles/r02b)
    int ffn_coop = 1;      // cooperative launch of the fused FFN (co-residency guaranteed; CASCADE_FFN_COOP=0: plain launch)
    float4* partial2 = nullptr;  // the fused kernel's down-phase partials / counters
    int* counters2 = nullptr;
    int* ffn_ready = nullptr;    // [slots] published gate/up super-tiles
    int invariant = 0;     // batch-invariant expert GEMV split (bitwise-lossless speculation)
    int* sm_index = nullptr;   // %smid -> dense SM index (SM-weighted expert GEMV split), nullptr: off
    int* sm_slot = nullptr;
    int* sm_cum = nullptr;     // [gemv_grid + 1]
    std::vector<float> sm_weight;  // per dense SM (host copy, diagnostics)
    int* attn_arrive = nullptr;
    int qkv_cluster = 0;   // cluster size of the split-K QKV GEMV (0: stream-K path)
    int pf_o = 0;          // attention CTAs (the whole grid) bulk-prefetch W_o into L2 after their wait
    int umma_no_trigger = 0;  // A/B: tcgen05 GEMVs let their dependents launch only at exit
    int pf_self = 0;       // cluster GEMVs bulk-prefetch the rest of their k-range into L2 before their wait (mask: 1 QKV, 2 O)
    int dense_pf = 0;      // tcgen05 GEMVs: rolling L2 prefetch this many ring stages ahead (CASCADE_DENSE_PF)
    int cluster_stages = kUStages;  // ring depth of the split-K O projection
    int o_cluster = 0;     // same for the O projection
    int qkv_stages = 3;    // QKV ring: 3 stages of 16 k-steps (64 KB of weights each; A/B in DESIGN §4)
    int qkv_stage_ks = kCMaxStageKs;
    int dn_prefetch = 8;   // fused FFN: k-steps of each warp's down range prefetched to L2 during the readiness wait (A/B: -1.5% at K=0)
    int min_seg = 8;       // k-steps per warp below which the stream-K split uses fewer pieces than CTAs
    int par_topk = 1;      // router top-k by parallel rank counting (CASCADE_TOPK_PAR=0: k serial warp selections)
    uint16_t* kc = nullptr;
    uint16_t* vc = nullptr;
    float* logits_full = nullptr;  // taps only
    cudaGraphExec_t graph[kMaxT + 1] = {};
    int graph_kernels[kMaxT + 1] = {};
    bool taps_on = false;
    Taps taps;
    int gemv_grid = 0;
    double t_base_ns = 0.0;
};

template <typename T>
static int salloc(cascade_session* s, T** p, size_t bytes, bool zero = true) {
    void* v = nullptr;
    CK(cudaMalloc(&v, bytes));
    s->allocs.push_back(v);
    if (zero) CK(cudaMemset(v, 0, bytes));
    *p = (T*)v;
    return CASCADE_OK;
}

extern "C" int cascade_session_destroy(cascade_session* s) {
    if (!s) return CASCADE_OK;
    cudaSetDevice(s->m->device);
    cudaStreamSynchronize(s->stream);
    for (auto& g : s->graph)
        if (g) cudaGraphExecDestroy(g);
    for (void* p : s->allocs) cudaFree(p);
    if (s->h_params) cudaFreeHost(s->h_params);
    if (s->h_result) cudaFreeHost(s->h_result);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
    return CASCADE_OK;
}

// SM-weighted split of the expert GEMVs (see sm_rate_probe_kernel).  Only
// when the GEMV occupancy is exactly 2 CTAs per SM (the work index relies
// on it) and the weights are large enough for a meaningful probe.
static int calibrate_sm_rates(cascade_session* s) {
    cascade_model* m = s->m;
    const Dims D(m->g);
    // measured: the CTA exit spread did not shrink and both expert GEMVs got
    // 2-4% slower (profiles/r01d/ab_sm_weights.txt), so it is opt-in
    const char* v = getenv("CASCADE_SM_WEIGHTS");
    if (!v || v[0] != '1') return CASCADE_OK;
    int occ1 = 0, occ2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, stream_gemv_kernel<1, EPI_GATEUP>, kGemvThreads,
                                                      gemv_smem_bytes<1>()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, stream_gemv_kernel<2, EPI_DOWN>, kGemvThreads,
                                                      gemv_smem_bytes<2>()) != cudaSuccess) {
        cudaGetLastError();
        return CASCADE_OK;
    }
    int occp = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occp, sm_rate_probe_kernel, kGemvThreads, 0);
    if (occ1 != 2 || occ2 != 2 || occp < 2 || s->gemv_grid != 2 * m->num_sms || m->layers.empty()) return CASCADE_OK;
    for (int t = 0; t < 5; ++t) {  // the other instantiations must be 2 per SM as well
        const void* k[5] = {(const void*)stream_gemv_kernel<1, EPI_STORE>, (const void*)stream_gemv_kernel<1, EPI_DOWN>,
                            (const void*)stream_gemv_kernel<2, EPI_GATEUP>, (const void*)stream_gemv_kernel<2, EPI_STORE>,
                            (const void*)stream_gemv_kernel<1, EPI_ARGMAX>};
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k[t], kGemvThreads, t < 2 || t == 4 ? gemv_smem_bytes<1>() : gemv_smem_bytes<2>());
        if (o != 2) return CASCADE_OK;
    }
    const int grid = s->gemv_grid;
    const long long avail_vec = (long long)m->n_blocks * D.w13_vec;
    long long per_cta = std::min<long long>(avail_vec / grid, (4ll << 20) / 16);
    if (per_cta * 16 < (256 << 10)) return CASCADE_OK;  // too little to time
    unsigned long long* d_out = nullptr;
    if (cudaMalloc(&d_out, (size_t)grid * 2 * 8) != cudaSuccess) {
        cudaGetLastError();
        return CASCADE_OK;
    }
    std::vector<unsigned long long> h((size_t)grid * 2);
    std::vector<double> dur(256, 0.0);
    std::vector<int> cnt(256, 0);
    const int reps = 7;
    bool ok = true;
    for (int r = 0; r < reps && ok; ++r) {
        sm_rate_probe_kernel<<<grid, kGemvThreads, 0, s->stream>>>(m->layers[0].w13, per_cta, d_out);
        ok = cudaStreamSynchronize(s->stream) == cudaSuccess &&
             cudaMemcpy(h.data(), d_out, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess;
        if (!ok || r == 0) continue;  // first run warms up
        for (int b = 0; b < grid; ++b) {
            const int smid = (int)(h[2 * b] & 0xFF);
            dur[smid] += (double)h[2 * b + 1];
            cnt[smid] += 1;
        }
    }
    cudaFree(d_out);
    if (!ok) {
        cudaGetLastError();
        return CASCADE_OK;
    }
    std::vector<int> index(256, -1);
    std::vector<double> rate;
    for (int smid = 0; smid < 256; ++smid) {
        if (cnt[smid] == 0) continue;
        if (cnt[smid] != 2 * (reps - 1)) return CASCADE_OK;  // not exactly 2 CTAs per SM: keep the equal split
        index[smid] = (int)rate.size();
        rate.push_back(cnt[smid] / dur[smid]);
    }
    if ((int)rate.size() * 2 != grid) return CASCADE_OK;
    double mean = 0.0;
    for (double r : rate) mean += r;
    mean /= rate.size();
    s->sm_weight.assign(rate.size(), 1.0f);
    std::vector<double> w(grid);
    for (size_t i = 0; i < rate.size(); ++i) {
        const double wi = std::min(1.2, std::max(0.8, rate[i] / mean));
        s->sm_weight[i] = (float)wi;
        w[2 * i] = w[2 * i + 1] = std::round(wi * 256.0) / 256.0;  // quantised: a stable split for the session
    }
    double tot = 0.0;
    for (double x : w) tot += x;
    std::vector<int> cum(grid + 1);
    double acc = 0.0;
    for (int i = 0; i <= grid; ++i) {
        cum[i] = (int)std::llround(acc / tot * (double)(1 << 24));
        if (i < grid) acc += w[i];
    }
    cum[grid] = 1 << 24;
    int rc;
    if ((rc = salloc(s, &s->sm_index, 256 * 4)) || (rc = salloc(s, &s->sm_slot, 256 * 4)) ||
        (rc = salloc(s, &s->sm_cum, (size_t)(grid + 1) * 4)))
        return rc;
    CK(cudaMemcpy(s->sm_index, index.data(), 256 * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s->sm_cum, cum.data(), (size_t)(grid + 1) * 4, cudaMemcpyHostToDevice));
    return CASCADE_OK;
}

extern "C" int cascade_session_create(cascade_model* m, int max_ctx, int k_max, void* stream,
                                      cascade_session** out) {
    if (!m || !out) return set_err(CASCADE_EINVAL, "model/out is NULL");
    if (max_ctx < 1) return set_err(CASCADE_EINVAL, "max_ctx must be >= 1");
    if (k_max < 0 || k_max > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "k_max must be in [0, 15]");
    CK(cudaSetDevice(m->device));
    cascade_session* s = new cascade_session();
    s->m = m;
    s->user_ctx = max_ctx;
    s->max_ctx = max_ctx + kMaxT;  // room for the in-flight rows
    s->k_max = k_max;
    s->max_chunks = (s->max_ctx + kChunk - 1) / kChunk + 1;
    if (s->max_chunks > kMaxChunksSmem) {
        delete s;
        return set_err(CASCADE_EINVAL, "max_ctx too large (limit 65000 positions)");
    }
    if (stream) {
        s->stream = (cudaStream_t)stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete s;
            return set_err(CASCADE_ECUDA, cudaGetErrorString(e));
        }
        s->own_stream = true;
    }
    const Dims D(m->g);
    const int G = D.H / D.KV;
    const int nslots = m->n_blocks;
    s->gemv_grid = m->num_sms * 2;
    const long long workers = (long long)s->gemv_grid * kGemvWarps;
    long long max_units = std::max<long long>({(long long)D.qkvd / kSTRows, (long long)D.d / kSTRows,
                                               (long long)nslots * (2 * D.f) / kSTRows,
                                               (long long)nslots * D.d / kSTRows, (long long)D.V / kSTRows});
    int rc;
    auto fail = [&](int code) {
        std::string msg = g_err;
        cascade_session_destroy(s);
        g_err = msg;
        return code;
    };
    if ((rc = salloc(s, &s->d_params, sizeof(StepParams))) || (rc = salloc(s, &s->d_state, sizeof(DevState))) ||
        (rc = salloc(s, &s->d_result, sizeof(cascade_verify_out))) ||
        (rc = salloc(s, &s->x, (size_t)kMaxT * D.d * 4)) || (rc = salloc(s, &s->xn, (size_t)D.d * 32)) ||
        (rc = salloc(s, &s->xn_u, (size_t)D.d * 32)) ||
        (rc = salloc(s, &s->upartial, (size_t)m->num_sms * 2 * kUPartialFloats * 4, false)) ||
        (rc = salloc(s, &s->ucounters, (size_t)std::max({D.qkvd, D.d, D.V}) / kURows * 4)) ||
        (rc = salloc(s, &s->qkv, (size_t)kMaxT * D.qkvd * 4)) ||
        (rc = salloc(s, &s->attn_part, (size_t)D.KV * G * kMaxT * s->max_chunks * (D.hd + 2) * 4)) ||
        (rc = salloc(s, &s->attn_out, (size_t)D.hq * 32)) ||
        (rc = salloc(s, &s->logits_router, (size_t)kMaxT * (D.E + 1) * 4)) ||
        (rc = salloc(s, &s->topk_id, (size_t)kMaxT * D.k * 4)) ||
        (rc = salloc(s, &s->topk_w, (size_t)kMaxT * D.k * 4)) || (rc = salloc(s, &s->gsh, kMaxT * 4)) ||
        (rc = salloc(s, &s->list, (size_t)(nslots + 1) * 4)) || (rc = salloc(s, &s->count, 4)) ||
        (rc = salloc(s, &s->route_rank, (size_t)(nslots + 1) * kMaxT * 4)) ||
        (rc = salloc(s, &s->union_size, (size_t)D.L * 4)) ||
        (rc = salloc(s, &s->hbuf, (size_t)std::max(nslots, 1) * D.f * 32)) ||
        (rc = salloc(s, &s->ycontrib, (size_t)kMaxT * (D.k + D.S) * D.d * 4)) ||
        (rc = salloc(s, &s->partial, (size_t)std::max<long long>(workers, (long long)nslots * s->gemv_grid) * 2 * kTPW * 2 * 32 * 16, false)) ||
        (rc = salloc(s, &s->partial2, (size_t)std::max<long long>(workers, (long long)nslots * s->gemv_grid) * 2 * kTPW * 2 * 32 * 16, false)) ||
        (rc = salloc(s, &s->counters2, (size_t)max_units * 4)) || (rc = salloc(s, &s->ffn_ready, (size_t)(nslots + 1) * kReadyStride * 4)) ||
        (rc = salloc(s, &s->counters, (size_t)max_units * 4)) || (rc = salloc(s, &s->attn_arrive, (size_t)D.KV * 4)) || (rc = salloc(s, &s->keys, kMaxT * 8)) ||
        (rc = salloc(s, &s->stamps, (size_t)(2 * D.L + 4) * 8)) || (rc = salloc(s, &s->tokens_used, kMaxT * 4)) ||
        (rc = salloc(s, &s->rope, (size_t)kMaxT * (D.hd / 2) * sizeof(float2))) ||
        (rc = salloc(s, &s->trace, 2048 * 8)) ||
        (rc = salloc(s, &s->kc, (size_t)D.L * D.KV * s->max_ctx * D.hd * 2, false)) ||
        (rc = salloc(s, &s->vc, (size_t)D.L * D.KV * s->max_ctx * D.hd * 2, false)))
        return fail(rc);
    cudaError_t e = cudaHostAlloc(&s->h_params, sizeof(StepParams) * (kMaxT + 1), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&s->h_result, sizeof(cascade_verify_out), cudaHostAllocDefault);
    if (e != cudaSuccess) {
        set_err(CASCADE_ECUDA, cudaGetErrorString(e));
        return fail(CASCADE_ECUDA);
    }
    std::memset(s->h_params, 0, sizeof(StepParams) * (kMaxT + 1));
    std::memset(s->h_result, 0, sizeof(cascade_verify_out));
    // Bulk L2 prefetch from latency-bound kernels measured slower on B200
    // (the issuing kernels stall on the bulk-prefetch queue); off by default.
    s->prefetch = false;
    if (const char* v = getenv("CASCADE_L2_PREFETCH")) s->prefetch = v[0] == '1';
    if (const char* v = getenv("CASCADE_PF_O")) s->pf_o = v[0] == '1';
    if (const char* v = getenv("CASCADE_PF_SELF")) s->pf_self = atoi(v) & 3;
    if (const char* v = getenv("CASCADE_DENSE_PF")) s->dense_pf = std::max(0, atoi(v));
    if (const char* v = getenv("CASCADE_UMMA_TRIGGER")) s->umma_no_trigger = v[0] == '0';
    if (const char* v = getenv("CASCADE_L2_PROLOGUE")) s->l2_prologue = atoi(v);  // 1: whole range, n > 1: first n k-steps
    if (const char* v = getenv("CASCADE_GEMV_TRIGGER")) s->gemv_trigger = v[0] == '1';
    if (const char* v = getenv("CASCADE_DOWN_EARLY")) s->down_early = v[0] == '1';
    if (const char* v = getenv("CASCADE_UMMA_PROLOGUE")) s->umma_prologue = v[0] == '1';
    if (const char* v = getenv("CASCADE_ATTN_FUSED")) s->attn_fused = v[0] == '1';
    if (const char* v = getenv("CASCADE_FFN_FUSED")) s->ffn_fused = v[0] == '1';
    if (const char* v = getenv("CASCADE_FFN_TRIGGER")) s->ffn_trigger = v[0] == '1';
    if (const char* v = getenv("CASCADE_FFN_COOP")) s->ffn_coop = v[0] == '1';
    if (const char* v = getenv("CASCADE_FFN_FMA")) s->ffn_fma = v[0] == '1';
    if (const char* v = getenv("CASCADE_FFN_RING")) s->ffn_ring = v[0] == '1';
    if (const char* v = getenv("CASCADE_RING_UNIT")) s->ring_unit_pieces = v[0] == '1';
    if (const char* v = getenv("CASCADE_RING_DNPF")) s->ring_dn_l2 = std::max(0, atoi(v));
    if (const char* v = getenv("CASCADE_RING_SLOTMAJOR")) s->ring_slot_major = v[0] == '1';
    if (const char* v = getenv("CASCADE_ATTN_KSPLIT")) s->attn_ksplit = std::max(0, std::min(3, atoi(v)));
    if (const char* v = getenv("CASCADE_RING_MAXT")) s->ring_max_t = std::max(0, std::min(kMaxT, atoi(v)));
    if (const char* v = getenv("CASCADE_UNIT_PIECES")) s->unit_pieces = v[0] == '1';
    if (const char* v = getenv("CASCADE_MIN_SEG")) s->min_seg = std::max(1, atoi(v));
    if (const char* v = getenv("CASCADE_TOPK_PAR")) s->par_topk = v[0] == '1';
    if (const char* v = getenv("CASCADE_DN_PF")) s->dn_prefetch = std::max(0, atoi(v));
    if (const char* v = getenv("CASCADE_INVARIANT")) s->invariant = v[0] == '1';
    if (const char* v = getenv("CASCADE_CLUSTER_STAGES")) s->cluster_stages = std::max(2, std::min(kCMaxStages, atoi(v)));
    if (const char* v = getenv("CASCADE_QKV_STAGE_KS")) s->qkv_stage_ks = std::max(1, std::min(kCMaxStageKs, atoi(v)));
    if (const char* v = getenv("CASCADE_QKV_STAGES")) s->qkv_stages = std::max(2, std::min(kCMaxStages, atoi(v)));
    if (dense_cluster_smem_bytes(s->qkv_stages, s->qkv_stage_ks) > 227 * 1024) {  // an override that does not fit
        s->qkv_stages = kUStages;
        s->qkv_stage_ks = kUStageKs;
    }
    if (const char* v = getenv("CASCADE_LATE_TRIGGER")) {
        const int late = (v[0] == '1' && v[1] == 0) ? 31 : atoi(v);  // "1": every latency-bound kernel; else a kLate* mask
        cudaMemcpyToSymbol(g_late_trigger, &late, sizeof(late));
    }
    // attention smem opt-in
    const int asmem = D.hd == 32 ? attn_smem_bytes<32>() : D.hd == 64 ? attn_smem_bytes<64>() : attn_smem_bytes<128>();
    if (D.hd == 32) e = cudaFuncSetAttribute(attn_partial_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, asmem);
    else if (D.hd == 64) e = cudaFuncSetAttribute(attn_partial_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, asmem);
    else e = cudaFuncSetAttribute(attn_partial_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, asmem);
    if (e == cudaSuccess) e = set_carveouts(D.hd);
    if (const char* v = getenv("CASCADE_ROUTE_STAGE")) g_route_stage = atoi(v);
    if (const char* v = getenv("CASCADE_ROUTE_CLUSTER")) g_route_cluster = atoi(v);
    (void)0;
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(moe_route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)route_smem_bytes(D, m->g.shared_gate));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_umma_smem_bytes());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_umma_smem_bytes());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_ARGMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_umma_smem_bytes());
    if (e == cudaSuccess) e = gemv_smem_attr<1>();
    if (e == cudaSuccess) e = gemv_smem_attr<2>();
    if (e == cudaSuccess) e = cudaFuncSetAttribute(expert_ffn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_smem_bytes<1>());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(expert_ffn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_smem_bytes<2>());
    if (e == cudaSuccess) e = carve(expert_ffn_kernel<1>);
    if (e == cudaSuccess) e = carve(expert_ffn_kernel<2>);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(expert_ffn_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, gemv_smem_bytes<1>());
    if (e == cudaSuccess) e = carve(expert_ffn_kernel<1, true>);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(expert_ffn_ring_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ffn_ring_smem_bytes<1>());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(expert_ffn_ring_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ffn_ring_smem_bytes<2>());
    if (e == cudaSuccess) e = carve(expert_ffn_ring_kernel<1>);
    if (e == cudaSuccess) e = carve(expert_ffn_ring_kernel<2>);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dense_gemv_cluster_kernel<UEPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   std::max(dense_cluster_smem_bytes(s->cluster_stages), dense_cluster_smem_bytes(s->qkv_stages, s->qkv_stage_ks)));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(dense_gemv_cluster_kernel<UEPI_ADD>, cudaFuncAttributeMaxDynamicSharedMemorySize, dense_cluster_smem_bytes(s->cluster_stages));
    if (const char* v = getenv("CASCADE_CLUSTER_STAGES")) s->cluster_stages = std::max(2, std::min(kCMaxStages, atoi(v)));
    if (e == cudaSuccess) e = carve(dense_gemv_cluster_kernel<UEPI_STORE>);
    if (e == cudaSuccess) e = carve(dense_gemv_cluster_kernel<UEPI_ADD>);
    if (e == cudaSuccess) {
        bool on = true;
        if (const char* v = getenv("CASCADE_DENSE_CLUSTER")) on = v[0] == '1';
        if (on && m->umma_qkv()) s->qkv_cluster = pick_cluster(m, D.qkvd / kURows, dense_cluster_smem_bytes(s->qkv_stages, s->qkv_stage_ks));
        if (on && m->umma_o()) s->o_cluster = pick_cluster(m, D.d / kURows, dense_cluster_smem_bytes(s->cluster_stages));
    }
    if (e != cudaSuccess) {
        set_err(CASCADE_ECUDA, cudaGetErrorString(e));
        return fail(CASCADE_ECUDA);
    }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        set_err(CASCADE_ECUDA, cudaGetErrorString(e));
        return fail(CASCADE_ECUDA);
    }
    // The fused FFN needs its whole grid (2 CTAs per SM) resident at once.
    // If this context cannot hold 2 per SM (a carveout override, an
    // SM-limited context), use the two-launch path, which has no
    // cross-CTA waits.
    if (s->ffn_fused) {
        int o1 = 0, o2 = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, expert_ffn_kernel<1>, kGemvThreads, gemv_smem_bytes<1>()) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, expert_ffn_kernel<2>, kGemvThreads, gemv_smem_bytes<2>()) != cudaSuccess) {
            cudaGetLastError();
            o1 = o2 = 0;
        }
        if (s->ffn_ring) {
            int r1 = 0, r2 = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r1, expert_ffn_ring_kernel<1>, ffn_ring_threads<1>(), ffn_ring_smem_bytes<1>()) != cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r2, expert_ffn_ring_kernel<2>, ffn_ring_threads<2>(), ffn_ring_smem_bytes<2>()) != cudaSuccess) {
                cudaGetLastError();
                r1 = r2 = 0;
            }
            if (std::min(r1, r2) < 1 || s->gemv_grid != 2 * m->num_sms) s->ffn_ring = 0;
        }
        if ((long long)std::min(o1, o2) * m->num_sms < s->gemv_grid) s->ffn_fused = 0;
    }
    if ((rc = calibrate_sm_rates(s))) return fail(rc);
    *out = s;
    return CASCADE_OK;
}

extern "C" void* cascade_session_stream(cascade_session* s) { return s ? (void*)s->stream : nullptr; }
extern "C" int cascade_session_geometry(cascade_session* s, cascade_geometry* out) {
    if (!s || !out) return set_err(CASCADE_EINVAL, "session/out is NULL");
    *out = s->m->g;
    return CASCADE_OK;
}
extern "C" int cascade_internal_vocab(const cascade_session* s) { return s ? s->m->g.vocab : 0; }

// ------------------------------------------------------------ step enqueue
// Every kernel of the step is launched with programmatic stream
// serialisation (PDL): it may be scheduled while its predecessor drains and
// blocks in griddepcontrol.wait until the predecessor's memory is visible.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int NT>
static cudaError_t launch_gemv_nt(int epi, const GemvParams& p, int grid, cudaStream_t st, bool pdl) {
    const size_t sm = gemv_smem_bytes<NT>();
    switch (epi) {
    case EPI_STORE: return launch_k(stream_gemv_kernel<NT, EPI_STORE>, grid, kGemvThreads, sm, st, pdl, p);
    case EPI_ADD: return launch_k(stream_gemv_kernel<NT, EPI_ADD>, grid, kGemvThreads, sm, st, pdl, p);
    case EPI_GATEUP: return launch_k(stream_gemv_kernel<NT, EPI_GATEUP>, grid, kGemvThreads, sm, st, pdl, p);
    case EPI_DOWN: return launch_k(stream_gemv_kernel<NT, EPI_DOWN>, grid, kGemvThreads, sm, st, pdl, p);
    default: return launch_k(stream_gemv_kernel<NT, EPI_ARGMAX>, grid, kGemvThreads, sm, st, pdl, p);
    }
}
// The fused expert FFN's down phase waits on gate/up tiles produced by other
// CTAs of the same grid, so the whole grid must be resident at once.  It is
// launched cooperatively: the driver then guarantees co-residency (or fails
// the launch with cudaErrorCooperativeLaunchTooLarge) even when other
// sessions' kernels share the GPU, instead of relying on an idle device.
static cudaError_t launch_ffn(const FfnParams& f, int grid, cudaStream_t st, bool coop, bool fma, bool ring) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ring ? grid / 2 : grid);  // ring: one CTA per SM
    cfg.blockDim = dim3(ring ? (f.gu.T <= 8 ? ffn_ring_threads<1>() : ffn_ring_threads<2>()) : kGemvThreads);
    cfg.dynamicSmemBytes = ring ? (f.gu.T <= 8 ? ffn_ring_smem_bytes<1>() : ffn_ring_smem_bytes<2>())
                                : f.gu.T <= 8 ? gemv_smem_bytes<1>() : gemv_smem_bytes<2>();
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 2 : 1;
    if (ring) return f.gu.T <= 8 ? cudaLaunchKernelEx(&cfg, expert_ffn_ring_kernel<1>, f)
                                 : cudaLaunchKernelEx(&cfg, expert_ffn_ring_kernel<2>, f);
    if (fma && f.gu.T == 1) return cudaLaunchKernelEx(&cfg, expert_ffn_kernel<1, true>, f);
    if (f.gu.T <= 8) return cudaLaunchKernelEx(&cfg, expert_ffn_kernel<1>, f);
    return cudaLaunchKernelEx(&cfg, expert_ffn_kernel<2>, f);
}
static cudaError_t launch_gemv(int epi, const GemvParams& p, int grid, cudaStream_t st, bool pdl = true) {
    return p.T <= 8 ? launch_gemv_nt<1>(epi, p, grid, st, pdl) : launch_gemv_nt<2>(epi, p, grid, st, pdl);
}



// moe_route_kernel: one CTA (or a cluster of p.C CTAs) per token, PDL.
static cudaError_t launch_route(const RouteParams& p, int T, size_t smem, cudaStream_t st) {
    const int C = p.C > 1 ? p.C : 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(T * C);
    cfg.blockDim = dim3(kRowThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = C;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = C > 1 ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, moe_route_kernel, p);
}

static cudaError_t launch_ugemv(int epi, const UGemvParams& p, int grid, cudaStream_t st) {
    const size_t sm = gemv_umma_smem_bytes();
    switch (epi) {
    case UEPI_STORE: return launch_k(stream_gemv_umma_kernel<UEPI_STORE>, grid, kUThreads, sm, st, true, p);
    case UEPI_ADD: return launch_k(stream_gemv_umma_kernel<UEPI_ADD>, grid, kUThreads, sm, st, true, p);
    default: return launch_k(stream_gemv_umma_kernel<UEPI_ARGMAX>, grid, kUThreads, sm, st, true, p);
    }
}

static UGemvParams ugemv_base(cascade_session* s, int T) {
    UGemvParams p{};
    p.T = T;
    p.n_blocks = 1;
    p.partial = s->upartial;
    p.counters = s->ucounters;
    p.no_prologue = !s->umma_prologue;
    p.ring_stages = s->cluster_stages;
    p.stage_ks = kUStageKs;
    p.pf_self = s->pf_self;
    p.pf_ahead = s->dense_pf;
    p.no_trigger = s->umma_no_trigger;
    return p;
}

static GemvParams gemv_base(cascade_session* s, int T) {
    GemvParams p{};
    p.T = T;
    p.min_seg = s->min_seg;
    p.partial = s->partial;
    p.counters = s->counters;
    p.invariant = s->invariant;
    p.unit_pieces = s->unit_pieces;
    p.sm_index = s->sm_index;
    p.sm_slot = s->sm_slot;
    p.cum = s->sm_cum;
    p.n_blocks = 1;
    p.l2_prologue = s->l2_prologue;
    p.trigger = s->gemv_trigger;
    return p;
}

// Optional per-launch event pairs (cascade_profile_step).
struct Prof {
    std::vector<cudaEvent_t> ev;
    std::vector<int> kind;
    cudaStream_t st = nullptr;
    void begin(int k) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
        ev.push_back(a);
        ev.push_back(b);
        kind.push_back(k);
    }
    void end() { cudaEventRecord(ev.back(), st); }
    ~Prof() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};
#define PB(k) \
    if (prof) prof->begin(k)
#define PE() \
    if (prof) prof->end()

// Enqueues one full step of width T on s->stream; returns the number of
// kernels launched through *n_kernels.
static int enqueue_step(cascade_session* s, int T, int* n_kernels, Prof* prof = nullptr) {
    cascade_model* m = s->m;
    const Dims D(m->g);
    const cudaStream_t st = s->stream;
    const bool taps = s->taps_on;
    int nk = 0;
    int slot = 0;
    auto tr = [&](int kind) {
        s->trace_kind[T][slot] = kind;
        return s->trace + slot++;
    };
    const bool pf = s->prefetch;
    CK(cudaMemcpyAsync(s->d_params, s->h_params + T, sizeof(StepParams), cudaMemcpyHostToDevice, st));

    EmbedParams ep{};
    ep.sp = s->d_params;
    ep.st = s->d_state;
    ep.embed = m->embed;
    ep.norm_w = m->layers[0].attn_norm;
    ep.x = s->x;
    ep.xn_bfrag = m->umma_qkv() ? s->xn_u : s->xn;
    ep.umma = m->umma_qkv();
    ep.tokens_used = s->tokens_used;
    ep.stamp = s->stamps;
    ep.tap_x = taps ? s->taps.x_in : nullptr;
    ep.tap_xn = taps ? s->taps.xn_attn : nullptr;
    ep.rope = s->rope;
    ep.T = T;
    ep.d = D.d;
    ep.hd = D.hd;
    ep.rope_theta = (double)m->g.rope_theta;
    ep.eps = m->g.norm_eps;
    ep.pf = pf ? m->layers[0].wqkv : nullptr;
    ep.pf_bytes = pf ? D.wqkv_vec * 16 : 0;
    ep.trace = tr(0);
    PB(0);
    CK(launch_k(embed_norm_kernel, dim3(T), dim3(kRouteThreads), 0, st, false, ep));
    PE();
    ++nk;

    const int G = D.H / D.KV;
    for (int l = 0; l < D.L; ++l) {
        const LayerW& w = m->layers[l];
        const size_t td = (size_t)l * kMaxT * D.d;
        // QKV
        PB(1);
        if (m->umma_qkv()) {
            UGemvParams q = ugemv_base(s, T);
            q.W = reinterpret_cast<const uint16_t*>(w.wqkv);
            q.B = s->xn_u;
            q.n_st = D.qkvd / kURows;
            q.n_ks = D.d / 16;
            q.out = s->qkv;
            q.ld = D.qkvd;
            q.stamp = s->stamps + 1 + 2 * l;
            q.trace = tr(1);
            q.pf_self = s->pf_self & 1;
            q.ring_stages = s->qkv_stages;
            q.stage_ks = s->qkv_stage_ks;
            if (s->qkv_cluster) CK(launch_dense_cluster(UEPI_STORE, q, s->qkv_cluster, st));
            else CK(launch_ugemv(UEPI_STORE, q, m->num_sms, st));
        } else {
            GemvParams q = gemv_base(s, T);
            q.W = w.wqkv;
            q.B = reinterpret_cast<const uint2*>(s->xn);
            q.n_st = D.qkvd / kSTRows;
            q.n_ks = D.d / 16;
            q.out = s->qkv;
            q.ld = D.qkvd;
            q.stamp = s->stamps + 1 + 2 * l;
            q.trace = tr(1);
            CK(launch_gemv(EPI_STORE, q, s->gemv_grid, st));
        }
        PE();
        ++nk;
        // attention
        AttnParams ap{};
        ap.qkv = s->qkv;
        ap.kc = s->kc + (size_t)l * D.KV * s->max_ctx * D.hd;
        ap.vc = s->vc + (size_t)l * D.KV * s->max_ctx * D.hd;
        ap.ctx_ptr = &s->d_state->cache_len;
        ap.rope = s->rope;
        ap.part = s->attn_part;
        ap.T = T;
        ap.H = D.H;
        ap.KV = D.KV;
        ap.max_ctx = s->max_ctx;
        ap.max_chunks = s->max_chunks;
        ap.scale = 1.0f / sqrtf((float)D.hd);
        ap.pf = (pf || s->pf_o) ? w.wo : nullptr;
        ap.pf_bytes = (pf || s->pf_o) ? D.wo_vec * 16 : 0;
        ap.trace = tr(2);
        // smem sized for this T's query rows; as many CTAs per SM as fit the
        // carveout (items are (chunk, kv head): 272 for OLMoE at ctx 1024)
        const int qrows = (G * T + 15) / 16 * 16;
        const int asm_ = D.hd == 32 ? attn_smem_bytes<32>(qrows) : D.hd == 64 ? attn_smem_bytes<64>(qrows)
                                                                                : attn_smem_bytes<128>(qrows);
        int per_sm = 1;  // resident CTAs per SM for this smem size (registers can bind first)
        {
            cudaError_t oe = D.hd == 32 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_partial_kernel<32>, kAttnThreads, asm_)
                             : D.hd == 64 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_partial_kernel<64>, kAttnThreads, asm_)
                                          : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_partial_kernel<128>, kAttnThreads, asm_);
            if (oe != cudaSuccess || per_sm < 1) {
                cudaGetLastError();
                per_sm = 1;
            }
            per_sm = std::min(per_sm, 4);
        }
        const int agrid = m->num_sms * per_sm;
        // fused combine needs [R][chunks] + [R] floats of the kernel's smem
        // and is only worth it while one CTA can keep every load in flight
        // (one (row, 4-dim) item per thread); wider T use attn_combine
        // (and short contexts: the merge loads 9 chunk partials per round trip)
        const bool fused = s->attn_fused && ((long long)(G * T) * (2 * s->max_chunks + 1)) * 4 <= asm_ &&
                           G * T * (D.hd / 4) <= kAttnThreads && s->max_chunks <= 27;
        ap.fused = fused;
        ap.arrive = s->attn_arrive;
        ap.out_bfrag = s->attn_out;
        ap.umma = m->umma_o();
        {
            // mma per warp: key split 64 * ceil(R/16), transposed 32 * ceil(R/8)
            // in passes of 4 row tiles -> transposed when ceil(R/8) is 1 or 3
            const int nr = (G * T + 7) / 8;
            ap.ksplit = s->attn_ksplit == 3 ? ((nr == 1 || nr == 3) ? 2 : 1) : s->attn_ksplit;
        }
        PB(2);
        if (D.hd == 32) CK(launch_k(attn_partial_kernel<32>, agrid, kAttnThreads, asm_, st, true, ap));
        else if (D.hd == 64) CK(launch_k(attn_partial_kernel<64>, agrid, kAttnThreads, asm_, st, true, ap));
        else CK(launch_k(attn_partial_kernel<128>, agrid, kAttnThreads, asm_, st, true, ap));
        PE();
        ++nk;
        if (!fused) {
            AttnCombineParams cp{};
            cp.part = s->attn_part;
            cp.ctx_ptr = &s->d_state->cache_len;
            cp.out_bfrag = s->attn_out;
            cp.tap = nullptr;
            cp.T = T;
            cp.H = D.H;
            cp.KV = D.KV;
            cp.hd = D.hd;
            cp.max_chunks = s->max_chunks;
            cp.umma = m->umma_o();
            cp.trace = tr(3);
            PB(3);
            CK(launch_k(attn_combine_kernel, dim3(T, D.H), dim3(D.hd), 0, st, true, cp));
            PE();
            ++nk;
        }
        (void)G;
        // O projection + residual
        PB(4);
        if (m->umma_o()) {
            UGemvParams o = ugemv_base(s, T);
            o.W = reinterpret_cast<const uint16_t*>(w.wo);
            o.B = s->attn_out;
            o.n_st = D.d / kURows;
            o.n_ks = D.hq / 16;
            o.out = s->x;
            o.ld = D.d;
            o.trace = tr(4);
            o.pf_self = (s->pf_self >> 1) & 1;
            if (s->o_cluster) CK(launch_dense_cluster(UEPI_ADD, o, s->o_cluster, st));
            else CK(launch_ugemv(UEPI_ADD, o, m->num_sms, st));
        } else {
            GemvParams o = gemv_base(s, T);
            o.W = w.wo;
            o.B = reinterpret_cast<const uint2*>(s->attn_out);
            o.n_st = D.d / kSTRows;
            o.n_ks = D.hq / 16;
            o.out = s->x;
            o.ld = D.d;
            o.trace = tr(4);
            CK(launch_gemv(EPI_ADD, o, s->gemv_grid, st));
        }
        PE();
        ++nk;
        if (taps) CK(cudaMemcpyAsync(s->taps.x_mid + td, s->x, (size_t)T * D.d * 4, cudaMemcpyDeviceToDevice, st));
        // route: norm + router + top-k + union
        RouteParams rp{};
        rp.x = s->x;
        rp.norm_w = w.ffn_norm;
        rp.router_w = w.router;
        rp.xn_bfrag = s->xn;
        rp.logits = s->logits_router;
        rp.topk_id = s->topk_id;
        rp.topk_w = s->topk_w;
        rp.gsh = s->gsh;
        rp.ycontrib = s->ycontrib;
        rp.tap_xn = taps ? s->taps.xn_moe + td : nullptr;
        rp.T = T;
        rp.d = D.d;
        rp.E = D.E;
        rp.k = D.k;
        rp.S = D.S;
        rp.renorm = m->g.renormalize_topk;
        rp.shared_gate = m->g.shared_gate;
        rp.e_lo = m->e_lo;
        rp.e_hi = m->e_hi;
        rp.ep_rank = m->ep_rank;
        rp.ep_size = m->ep_size;
        rp.eps = m->g.norm_eps;
        rp.zero_nonlocal = m->ep_size > 1;
        rp.stage_w = route_staged(D, m->g.shared_gate);
        rp.C = route_cluster(D, m->g.shared_gate);
        rp.ffn_ready = s->ffn_fused ? s->ffn_ready : nullptr;
        rp.n_ready = m->n_blocks;
        rp.par_topk = s->par_topk;
        rp.stamp = s->stamps + 2 + 2 * l;
        rp.trace = tr(5);
        PB(5);
        CK(launch_route(rp, T, route_smem_bytes(D, m->g.shared_gate), st));
        PE();
        ++nk;
        if (getenv("CASCADE_ROUTE_TWICE")) {  // i-cache experiment
            rp.trace = tr(5);
            CK(launch_route(rp, T, route_smem_bytes(D, m->g.shared_gate), st));
            ++nk;
        }
        if (taps) {
            CK(cudaMemcpyAsync(s->taps.logits + (size_t)l * kMaxT * (D.E + 1), s->logits_router,
                               (size_t)T * (D.E + 1) * 4, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(s->taps.topk_id + (size_t)l * kMaxT * D.k, s->topk_id, (size_t)T * D.k * 4,
                               cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(s->taps.topk_w + (size_t)l * kMaxT * D.k, s->topk_w, (size_t)T * D.k * 4,
                               cudaMemcpyDeviceToDevice, st));
        }
        // experts: gate/up (+SiLU) then down, over the active list only
        auto set_union = [&](GemvParams& q) {
            q.topk_id = s->topk_id;
            q.k_top = D.k;
            q.E = D.E;
            q.e_lo = m->e_lo;
            q.e_hi = m->e_hi;
            q.S = D.S;
            q.ep_rank = m->ep_rank;
            q.ep_size = m->ep_size;
        };
        GemvParams gu = gemv_base(s, T);
        gu.W = w.w13;
        gu.w_block_stride = D.w13_vec;
        gu.B = reinterpret_cast<const uint2*>(s->xn);
        gu.b_block_stride = 0;
        gu.list = s->list;    // published union (CTA 0): accept, telemetry, taps
        gu.count = s->count;
        gu.route_rank = s->route_rank;
        gu.union_size = s->union_size + l;
        gu.publish = 1;
        set_union(gu);
        gu.n_st = 2 * D.f / kSTRows;
        gu.n_ks = D.d / 16;
        gu.hout = s->hbuf;
        gu.h_block_stride = (long long)D.f * 16;
        gu.trace = tr(6);
        GemvParams dn = gemv_base(s, T);
        dn.W = w.w2;
        dn.w_block_stride = D.w2_vec;
        dn.B = reinterpret_cast<const uint2*>(s->hbuf);
        dn.b_block_stride = (long long)D.f * 4;  // uint2 units per slot
        set_union(dn);
        dn.n_st = D.d / kSTRows;
        dn.n_ks = D.f / 16;
        dn.early_list = s->down_early;  // union from the router's top-k, written two kernels back
        dn.n_contrib = D.k + D.S;
        dn.out = s->ycontrib;
        dn.ld = D.d;
        if (s->ffn_fused) {
            FfnParams fp{};
            fp.gu = gu;
            fp.dn = dn;
            fp.dn.partial = s->partial2;
            fp.dn.trace = gu.trace;  // per-CTA phase stamps of the down phase (diagnostic trace only)
            fp.dn.l2_prologue = s->dn_prefetch;
            fp.dn.counters = s->counters2;
            fp.ready = s->ffn_ready;
            fp.n_st_gu = gu.n_st;
            fp.dn_l2_stages = s->ring_dn_l2;
            // dependents launch at exit: an early-resident combine CTA made
            // its own loads 2x slower (A/B, profiles/r01f/ab_ffn_trigger.txt)
            fp.gu.trigger = s->ffn_trigger;
            PB(6);
            // CUDA-core single-token engine only outside batch-invariant mode (it
            // would give the pending token other sums at K = 0 than at K > 0)
            // ring engine (one TMA stream per SM) for up to 8 tokens; with more
            // the token block no longer fits L1 and the register engine is
            // faster (A/B in profiles/r02b).  Batch-invariant mode keeps one
            // engine for every T.
            const bool ring = s->ffn_ring && !s->invariant && T <= s->ring_max_t;
            if (ring && s->ring_slot_major) {
                // Slot-major pieces: every CTA streams its 1/grid of slot 0's
                // gate/up, then of slot 1's, ..., then the same for down, so
                // slot b's gate/up is complete chip-wide long before any CTA
                // reaches slot b's down: no gate/up -> down readiness wait.
                // Only for experts large enough that a slot's piece per CTA
                // is >= min_seg k-steps per warp (P == grid for both phases).
                auto pieces = [&](long long per_block) {
                    long long pm = per_block / ((long long)s->min_seg * kGemvWarps);
                    return pm < s->gemv_grid / 2 ? pm : (long long)(s->gemv_grid / 2);
                };
                const int g1 = s->gemv_grid / 2;
                if (pieces((long long)gu.n_st * gu.n_ks) == g1 && pieces((long long)dn.n_st * dn.n_ks) == g1) {
                    fp.gu.invariant = 1;
                    fp.dn.invariant = 1;
                }
            }
            if (ring && !s->ring_unit_pieces) {
                // one CTA per SM: whole super-tiles per CTA would idle SMs, and the
                // ring finalises the two boundary super-tiles of a piece off the
                // critical path anyway
                fp.gu.unit_pieces = 0;
                fp.dn.unit_pieces = 0;
            }
            CK(launch_ffn(fp, s->gemv_grid, st, s->ffn_coop, s->ffn_fma && !s->invariant, ring));
            PE();
            ++nk;
        } else {
            PB(6);
            CK(launch_gemv(EPI_GATEUP, gu, s->gemv_grid, st));
            PE();
            ++nk;
            dn.trace = tr(7);
            PB(7);
            CK(launch_gemv(EPI_DOWN, dn, s->gemv_grid, st));
            PE();
            ++nk;
        }
        if (m->comm) {
            PB(11);
            const int nr = g_nccl.AllReduce(s->ycontrib, s->ycontrib, (size_t)T * (D.k + D.S) * D.d, kNcclFloat32,
                                            kNcclSum, m->comm, st);
            PE();
            if (nr != 0) return set_err(CASCADE_ERUNTIME, "ncclAllReduce failed");
        }
        CombineParams c{};
        c.x = s->x;
        c.ycontrib = s->ycontrib;
        c.topk_w = s->topk_w;
        c.gsh = s->gsh;
        c.norm_w = (l + 1 < D.L) ? m->layers[l + 1].attn_norm : m->final_norm;
        {
            const bool next_umma = (l + 1 < D.L) ? m->umma_qkv() : m->umma_lm();
            c.xn_bfrag = next_umma ? s->xn_u : s->xn;
            c.umma = next_umma;
        }
        c.tap_moe = taps ? s->taps.moe_out + td : nullptr;
        c.tap_xn = (taps && l + 1 < D.L) ? s->taps.xn_attn + td + (size_t)kMaxT * D.d : nullptr;
        c.tap_x = (taps && l + 1 < D.L) ? s->taps.x_in + td + (size_t)kMaxT * D.d : nullptr;
        c.T = T;
        c.d = D.d;
        c.k = D.k;
        c.S = D.S;
        c.eps = m->g.norm_eps;
        c.pf = (pf && l + 1 < D.L) ? m->layers[l + 1].wqkv : nullptr;
        c.pf_bytes = (pf && l + 1 < D.L) ? D.wqkv_vec * 16 : 0;
        c.trace = tr(8);
        PB(8);
        CK(launch_k(moe_combine_kernel, dim3(T), dim3(kRowThreads), 0, st, m->comm == nullptr, c));
        PE();
        ++nk;
    }
    // LM head + argmax
    PB(9);
    if (m->umma_lm()) {
        UGemvParams lm = ugemv_base(s, T);
        lm.W = reinterpret_cast<const uint16_t*>(m->lm_head);
        lm.B = s->xn_u;
        lm.n_st = D.V / kURows;
        lm.n_ks = D.d / 16;
        lm.keys = s->keys;
        lm.out = taps ? s->taps.final_logits : nullptr;
        lm.ld = D.V;
        lm.stamp = s->stamps + 1 + 2 * D.L;
        lm.trace = tr(9);
        CK(launch_ugemv(UEPI_ARGMAX, lm, m->num_sms, st));
    } else {
        GemvParams lm = gemv_base(s, T);
        lm.W = m->lm_head;
        lm.B = reinterpret_cast<const uint2*>(s->xn);
        lm.n_st = D.V / kSTRows;
        lm.n_ks = D.d / 16;
        lm.keys = s->keys;
        lm.out = taps ? s->taps.final_logits : nullptr;
        lm.ld = D.V;
        lm.stamp = s->stamps + 1 + 2 * D.L;
        lm.trace = tr(9);
        CK(launch_gemv(EPI_ARGMAX, lm, s->gemv_grid, st));
    }
    PE();
    ++nk;
    AcceptParams ap{};
    ap.sp = s->d_params;
    ap.st = s->d_state;
    ap.keys = s->keys;
    ap.tokens_used = s->tokens_used;
    ap.stamps = s->stamps;
    ap.union_size = s->union_size;
    ap.res = s->d_result;
    ap.T = T;
    ap.L = D.L;
    ap.S = D.S;
    ap.trace = tr(10);
    s->trace_n[T] = slot;
    PB(10);
    CK(launch_k(accept_kernel, dim3(1), dim3(32), 0, st, true, ap));
    PE();
    ++nk;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(s->h_result, s->d_result, sizeof(cascade_verify_out), cudaMemcpyDeviceToHost, st));
    if (n_kernels) *n_kernels = nk;
    return CASCADE_OK;
}

static int ensure_graph(cascade_session* s, int T) {
    if (s->graph[T]) return CASCADE_OK;
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    int nk = 0;
    int rc = enqueue_step(s, T, &nk);
    cudaError_t e = cudaStreamEndCapture(s->stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return set_err(CASCADE_ECUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&s->graph[T], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return set_err(CASCADE_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    s->graph_kernels[T] = nk;
    return CASCADE_OK;
}

static int run_step(cascade_session* s, int T) {
    if (s->taps_on) return enqueue_step(s, T, nullptr);
    int rc = ensure_graph(s, T);
    if (rc) return rc;
    CK(cudaGraphLaunch(s->graph[T], s->stream));
    return CASCADE_OK;
}

// Writes the step parameters of width T into slot T.  A graph already
// enqueued for width T copies the slot when it runs, so a changed slot is
// only written after the stream drained; an unchanged one is left alone
// (back-to-back enqueues of the same step need no host sync).
static int set_params(cascade_session* s, int T, int mode, int commit, const int32_t* tokens, double draft_ns) {
    StepParams p;
    std::memset(&p, 0, sizeof(p));
    p.mode = mode;
    p.commit = commit;
    p.T = T;
    for (int i = 0; i < kMaxT; ++i) p.tokens[i] = tokens ? tokens[i] : 0;
    p.t_base_ns = s->t_base_ns;
    p.draft_ns = draft_ns;
    if (std::memcmp(&p, s->h_params + T, sizeof(p)) != 0) {
        CK(cudaStreamSynchronize(s->stream));
        s->h_params[T] = p;
    }
    return CASCADE_OK;
}

// A committing step of width T must keep the committed KV length within
// the session's max_ctx; checked before anything is launched.
static int check_room(cascade_session* s, int T) {
    if (s->len_hi + T > s->user_ctx)
        return set_err(CASCADE_ERUNTIME, "session KV cache is full (max_ctx reached): cache_len " +
                                             std::to_string(s->len_hi) + " + " + std::to_string(T) +
                                             " in-flight rows > max_ctx " + std::to_string(s->user_ctx));
    return CASCADE_OK;
}

extern "C" int cascade_profile_step(cascade_session* s, int K, double* ns, int32_t* kind, int cap, int* n) {
    if (!s || !ns || !kind || !n || K < 0 || K > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "bad arguments");
    CK(cudaSetDevice(s->m->device));
    CK(cudaStreamSynchronize(s->stream));
    const int T = K + 1;
    int rc = set_params(s, T, 0, 0, s->drafts, 0.0);
    if (rc) return rc;
    Prof prof;
    prof.st = s->stream;
    rc = enqueue_step(s, T, nullptr, &prof);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->stream));
    const int cnt = (int)prof.kind.size();
    if (cnt > cap) return set_err(CASCADE_EINVAL, "profile buffer too small: need " + std::to_string(cnt));
    for (int i = 0; i < cnt; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, prof.ev[2 * i], prof.ev[2 * i + 1]));
        ns[i] = (double)ms * 1.0e6;
        kind[i] = prof.kind[i];
    }
    *n = cnt;
    return CASCADE_OK;
}

extern "C" int cascade_step_trace(cascade_session* s, int K, double* ns, int32_t* kind, int cap, int* n) {
    if (!s || !ns || !kind || !n || K < 0 || K > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "bad arguments");
    if (s->taps_on) return set_err(CASCADE_EINVAL, "step trace needs the captured path (disable taps)");
    CK(cudaSetDevice(s->m->device));
    CK(cudaStreamSynchronize(s->stream));
    const int T = K + 1;
    int rc = set_params(s, T, 0, 0, s->drafts, 0.0);
    if (rc) return rc;
    rc = run_step(s, T);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->stream));
    const int cnt = s->trace_n[T];
    if (cnt > cap) return set_err(CASCADE_EINVAL, "trace buffer too small: need " + std::to_string(cnt));
    std::vector<unsigned long long> st(cnt + 1);
    CK(cudaMemcpy(st.data(), s->trace, (cnt + 1) * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < cnt; ++i) {
        ns[i] = (double)st[i + 1] - (double)st[i];
        kind[i] = s->trace_kind[T][i];
    }
    *n = cnt;
    return CASCADE_OK;
}

extern "C" int cascade_step_cta_trace(cascade_session* s, int K, uint64_t* out, int32_t* kind, int cap_slots,
                                      int* n_slots) {
    if (!s || !out || !kind || !n_slots || K < 0 || K > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "bad arguments");
    if (s->taps_on) return set_err(CASCADE_EINVAL, "CTA trace needs the captured path (disable taps)");
    CK(cudaSetDevice(s->m->device));
    const int T = K + 1;
    int rc = ensure_graph(s, T);
    if (rc) return rc;
    const int cnt = s->trace_n[T];
    if (cnt > cap_slots) return set_err(CASCADE_EINVAL, "trace buffer too small: need " + std::to_string(cnt));
    const size_t bytes = (size_t)cnt * kCtaTraceCap * kCtaRec * 8;
    unsigned long long* buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    unsigned long long* base = s->trace;
    CK(cudaMemcpyToSymbol(g_cta_trace_base, &base, sizeof(base)));
    CK(cudaMemcpyToSymbol(g_cta_trace, &buf, sizeof(buf)));
    rc = set_params(s, T, 0, 0, s->drafts, 0.0);
    if (rc == CASCADE_OK) rc = run_step(s, T);
    cudaError_t e = cudaStreamSynchronize(s->stream);
    unsigned long long* null = nullptr;
    cudaMemcpyToSymbol(g_cta_trace, &null, sizeof(null));
    if (rc == CASCADE_OK && e == cudaSuccess) e = cudaMemcpy(out, buf, bytes, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (rc) return rc;
    if (e != cudaSuccess) return set_err(CASCADE_ECUDA, cudaGetErrorString(e));
    for (int i = 0; i < cnt; ++i) kind[i] = s->trace_kind[T][i];
    *n_slots = cnt;
    return CASCADE_OK;
}

extern "C" int cascade_step_kernel_count(cascade_session* s, int K, int* out) {
    if (!s || !out || K < 0 || K > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "bad arguments");
    CK(cudaSetDevice(s->m->device));
    int rc = ensure_graph(s, K + 1);
    if (rc) return rc;
    *out = s->graph_kernels[K + 1];
    return CASCADE_OK;
}

extern "C" int cascade_session_reset(cascade_session* s) {
    if (!s) return set_err(CASCADE_EINVAL, "session is NULL");
    CK(cudaSetDevice(s->m->device));
    // stream-ordered: no device-wide synchronize that would also wait on
    // (and interleave with) other sessions' work from other host threads
    CK(cudaMemsetAsync(s->d_state, 0, sizeof(DevState), s->stream));
    CK(cudaStreamSynchronize(s->stream));
    s->len_hi = 0;
    return CASCADE_OK;
}

extern "C" int cascade_set_batch_invariant(cascade_session* s, int on) {
    if (!s) return set_err(CASCADE_EINVAL, "bad arguments");
    CK(cudaSetDevice(s->m->device));
    CK(cudaStreamSynchronize(s->stream));
    const int v = on ? 1 : 0;
    if (v == s->invariant) return CASCADE_OK;
    s->invariant = v;
    for (int T = 0; T <= kMaxT; ++T)  // graphs bake the GEMV parameters: recapture lazily
        if (s->graph[T]) {
            cudaGraphExecDestroy(s->graph[T]);
            s->graph[T] = nullptr;
        }
    return CASCADE_OK;
}

extern "C" int cascade_set_baseline(cascade_session* s, double t_base_ns) {
    if (!s) return set_err(CASCADE_EINVAL, "session is NULL");
    if (!(t_base_ns > 0.0)) return set_err(CASCADE_EINVAL, "set_baseline: t_base must be > 0");
    s->t_base_ns = t_base_ns;
    return CASCADE_OK;
}

static int read_state(cascade_session* s, DevState* out) {
    CK(cudaMemcpyAsync(out, s->d_state, sizeof(DevState), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return CASCADE_OK;
}

extern "C" int cascade_prefill(cascade_session* s, const int32_t* prompt, int n) {
    if (!s || !prompt) return set_err(CASCADE_EINVAL, "session/prompt is NULL");
    if (n < 1) return set_err(CASCADE_EINVAL, "prefill: need at least one token");
    CK(cudaSetDevice(s->m->device));
    DevState ds;
    int rc = read_state(s, &ds);
    if (rc) return rc;
    s->len_hi = ds.cache_len;
    if (ds.cache_len + n - 1 > s->user_ctx) return set_err(CASCADE_EINVAL, "prefill exceeds max_ctx");
    for (int i = 0; i < n; ++i)
        if (prompt[i] < 0 || prompt[i] >= s->m->g.vocab) return set_err(CASCADE_EINVAL, "token id out of range");
    int pos = 0;
    while (pos < n - 1) {
        const int T = std::min(kMaxT, n - 1 - pos);
        int32_t tok[kMaxT] = {};
        for (int i = 0; i < T; ++i) tok[i] = prompt[pos + i];
        if ((rc = set_params(s, T, 1, 1, tok, 0.0))) return rc;
        std::memcpy(s->drafts, tok, sizeof(tok));
        if ((rc = run_step(s, T))) return rc;
        s->len_hi += T;
        pos += T;
    }
    // on the session's (non-blocking) stream: a legacy-stream copy from
    // pageable memory may return before its DMA lands, and the next step on
    // this stream would not wait for it
    const int32_t last = prompt[n - 1];
    CK(cudaMemcpyAsync(&s->d_state->pending, &last, 4, cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return CASCADE_OK;
}

extern "C" int cascade_verify(cascade_session* s, const int32_t* draft, int K, double draft_ns,
                              cascade_verify_out* out) {
    if (!s || !out) return set_err(CASCADE_EINVAL, "session/out is NULL");
    if (K < 0 || K > s->k_max) return set_err(CASCADE_EINVAL, "verify: K must be in [0, k_max]");
    if (K > 0 && !draft) return set_err(CASCADE_EINVAL, "verify: draft is NULL");
    for (int i = 0; i < K; ++i)
        if (draft[i] < 0 || draft[i] >= s->m->g.vocab) return set_err(CASCADE_EINVAL, "draft token out of range");
    CK(cudaSetDevice(s->m->device));
    const int T = K + 1;
    int rc = check_room(s, T);
    if (rc) return rc;
    int32_t tok[kMaxT] = {};
    for (int i = 0; i < K; ++i) tok[i + 1] = draft[i];
    if ((rc = set_params(s, T, 0, 1, tok, draft_ns))) return rc;
    std::memcpy(s->drafts, tok, sizeof(tok));
    s->len_hi += T;
    rc = run_step(s, T);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->stream));
    *out = *s->h_result;
    s->len_hi = out->cache_len;
    return CASCADE_OK;
}

extern "C" int cascade_verify_enqueue(cascade_session* s, int K, int commit) {
    if (!s) return set_err(CASCADE_EINVAL, "session is NULL");
    if (K < 0 || K > CASCADE_MAX_K) return set_err(CASCADE_EINVAL, "K out of range");
    const int T = K + 1;
    int rc = commit ? check_room(s, T) : CASCADE_OK;
    if (rc) return rc;
    if ((rc = set_params(s, T, 0, commit ? 1 : 0, s->drafts, 0.0))) return rc;
    rc = run_step(s, T);
    if (rc == CASCADE_OK && commit) s->len_hi += T;
    return rc;
}

extern "C" int cascade_sync(cascade_session* s) {
    if (!s) return set_err(CASCADE_EINVAL, "session is NULL");
    DevState ds;
    int rc = read_state(s, &ds);
    if (rc) return rc;
    s->len_hi = ds.cache_len;
    return CASCADE_OK;
}

extern "C" int cascade_last_union_sizes(cascade_session* s, int32_t* out, int n) {
    if (!s || !out || n < s->m->g.num_layers) return set_err(CASCADE_EINVAL, "need num_layers ints");
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaMemcpy(out, s->union_size, (size_t)s->m->g.num_layers * 4, cudaMemcpyDeviceToHost));
    return CASCADE_OK;
}

// ---------------------------------------------------------------- taps
extern "C" int cascade_enable_taps(cascade_session* s, int enable) {
    if (!s) return set_err(CASCADE_EINVAL, "session is NULL");
    const Dims D(s->m->g);
    if (enable && !s->taps.x_in) {
        const size_t ld = (size_t)D.L * kMaxT;
        int rc;
        if ((rc = salloc(s, &s->taps.xn_moe, ld * D.d * 2)) || (rc = salloc(s, &s->taps.logits, ld * (D.E + 1) * 4)) ||
            (rc = salloc(s, &s->taps.topk_id, ld * D.k * 4)) || (rc = salloc(s, &s->taps.topk_w, ld * D.k * 4)) ||
            (rc = salloc(s, &s->taps.moe_out, ld * D.d * 4)) ||
            (rc = salloc(s, &s->taps.final_logits, (size_t)kMaxT * D.V * 4)) ||
            (rc = salloc(s, &s->taps.xn_attn, ld * D.d * 2)) || (rc = salloc(s, &s->taps.x_mid, ld * D.d * 4)) ||
            (rc = salloc(s, &s->taps.x_in, ld * D.d * 4)))
            return rc;
    }
    s->taps_on = enable != 0;
    return CASCADE_OK;
}

extern "C" int cascade_read_tap(cascade_session* s, int kind, void* out, size_t bytes) {
    if (!s || !out) return set_err(CASCADE_EINVAL, "session/out is NULL");
    if (!s->taps.x_in) return set_err(CASCADE_EINVAL, "taps are not enabled");
    const Dims D(s->m->g);
    const size_t ld = (size_t)D.L * kMaxT;
    const void* src = nullptr;
    size_t n = 0;
    switch (kind) {
    case 0: src = s->taps.xn_moe; n = ld * D.d * 2; break;
    case 1: src = s->taps.logits; n = ld * (D.E + 1) * 4; break;
    case 2: src = s->taps.topk_id; n = ld * D.k * 4; break;
    case 3: src = s->taps.topk_w; n = ld * D.k * 4; break;
    case 4: src = s->taps.moe_out; n = ld * D.d * 4; break;
    case 5: src = s->taps.final_logits; n = (size_t)kMaxT * D.V * 4; break;
    case 6: src = s->taps.xn_attn; n = ld * D.d * 2; break;
    case 7: src = s->taps.x_mid; n = ld * D.d * 4; break;
    case 8: src = s->taps.x_in; n = ld * D.d * 4; break;
    default: return set_err(CASCADE_EINVAL, "unknown tap kind");
    }
    if (bytes != n) return set_err(CASCADE_EINVAL, "tap size mismatch: expected " + std::to_string(n));
    CK(cudaSetDevice(s->m->device));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaMemcpy(out, src, n, cudaMemcpyDeviceToHost));
    return CASCADE_OK;
}

// ---------------------------------------------------------------- weights readback
__global__ void afrag_extract_kernel(const uint16_t* src, int n_ks, int row_phys0, int phys_step_mode, int nrows,
                                     int cols, uint16_t* dst, int umma) {
    // phys_step_mode: 0 = rows contiguous; 1 = gate rows; 2 = up rows (GATEUP layout)
    const long long n = (long long)nrows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int rr = (int)(i / cols), c = (int)(i % cols);
        if (umma) {
            dst[i] = src[umma_a_index((long long)row_phys0 + rr, c, n_ks)];
            continue;
        }
        int R;
        if (phys_step_mode == 0) R = row_phys0 + rr;
        else {
            const int j = row_phys0 + rr;
            R = (j / 8) * 16 + (phys_step_mode == 2 ? 8 : 0) + (j % 8);
        }
        const int st = R / kSTRows, it = (R % kSTRows) / 16, r = R % 16;
        const int s = c / 16, cc = c % 16;
        const int g = r % 8, t = (cc % 8) / 2;
        const int e = (cc / 8) * 4 + (r / 8) * 2 + (cc % 2);
        const int lane = g * 4 + t;
        dst[i] = src[((((long long)st * n_ks + s) * kTPW + it) * 32 + lane) * 8 + e];
    }
}

extern "C" int cascade_read_weight(cascade_model* m, int kind, int layer, int expert, int row0, int nrows,
                                   uint16_t* out) {
    if (!m || !out || nrows < 1 || row0 < 0) return set_err(CASCADE_EINVAL, "bad arguments");
    const Dims D(m->g);
    if ((kind != CASCADE_T_EMBED && kind != CASCADE_T_LM_HEAD && kind != CASCADE_T_FINAL_NORM) &&
        (layer < 0 || layer >= D.L))
        return set_err(CASCADE_EINVAL, "layer out of range");
    CK(cudaSetDevice(m->device));
    const uint16_t* plain = nullptr;
    int cols = D.d, rows_total = 0;
    const uint4* af = nullptr;
    int n_ks = 0, mode = 0, phys0 = row0;
    int umma = 0;
    switch (kind) {
    case CASCADE_T_EMBED: plain = m->embed; rows_total = D.V; break;
    case CASCADE_T_FINAL_NORM: plain = m->final_norm; rows_total = 1; break;
    case CASCADE_T_ATTN_NORM: plain = m->layers[layer].attn_norm; rows_total = 1; break;
    case CASCADE_T_FFN_NORM: plain = m->layers[layer].ffn_norm; rows_total = 1; break;
    case CASCADE_T_ROUTER: plain = m->layers[layer].router; rows_total = D.E; break;
    case CASCADE_T_SHARED_GATE:
        plain = m->layers[layer].router + (size_t)D.E * D.d; rows_total = m->g.shared_gate ? 1 : 0; break;
    case CASCADE_T_WQ: af = m->layers[layer].wqkv; rows_total = D.hq; n_ks = D.d / 16; umma = m->umma_qkv(); break;
    case CASCADE_T_WK:
        af = m->layers[layer].wqkv; rows_total = D.KV * D.hd; n_ks = D.d / 16; phys0 = D.hq + row0;
        umma = m->umma_qkv();
        break;
    case CASCADE_T_WV:
        af = m->layers[layer].wqkv; rows_total = D.KV * D.hd; n_ks = D.d / 16; phys0 = D.hq + D.KV * D.hd + row0;
        umma = m->umma_qkv();
        break;
    case CASCADE_T_WO:
        af = m->layers[layer].wo; rows_total = D.d; cols = D.hq; n_ks = D.hq / 16; umma = m->umma_o(); break;
    case CASCADE_T_LM_HEAD: af = m->lm_head; rows_total = D.V; n_ks = D.d / 16; umma = m->umma_lm(); break;
    case CASCADE_T_W_GATE:
    case CASCADE_T_W_UP:
    case CASCADE_T_W_DOWN: {
        int b = -1;
        if (expert >= m->e_lo && expert < m->e_hi) b = expert - m->e_lo;
        else if (expert >= D.E && expert < D.E + D.S && ((expert - D.E) % m->ep_size) == m->ep_rank) {
            int lb = 0;
            for (int s2 = 0; s2 < expert - D.E; ++s2) lb += (s2 % m->ep_size) == m->ep_rank;
            b = (m->e_hi - m->e_lo) + lb;
        }
        if (b < 0) return set_err(CASCADE_EINVAL, "expert is not held by this rank");
        if (kind == CASCADE_T_W_DOWN) {
            af = m->layers[layer].w2 + (size_t)b * D.w2_vec; rows_total = D.d; cols = D.f; n_ks = D.f / 16;
        } else {
            af = m->layers[layer].w13 + (size_t)b * D.w13_vec; rows_total = D.f; n_ks = D.d / 16;
            mode = kind == CASCADE_T_W_GATE ? 1 : 2;
        }
        break;
    }
    default: return set_err(CASCADE_EINVAL, "unknown tensor kind");
    }
    if (row0 + nrows > rows_total) return set_err(CASCADE_EINVAL, "rows out of range");
    const size_t n = (size_t)nrows * cols;
    if (plain) {
        CK(cudaMemcpy(out, plain + (size_t)row0 * cols, n * 2, cudaMemcpyDeviceToHost));
        return CASCADE_OK;
    }
    uint16_t* tmp = nullptr;
    CK(cudaMalloc(&tmp, n * 2));
    afrag_extract_kernel<<<256, 256>>>(reinterpret_cast<const uint16_t*>(af), n_ks, phys0, mode, nrows, cols, tmp,
                                       umma);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(out, tmp, n * 2, cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    if (e != cudaSuccess) return set_err(CASCADE_ECUDA, cudaGetErrorString(e));
    return CASCADE_OK;
}

extern "C" int cascade_read_kv(cascade_session* s, int layer, int which, int len, uint16_t* out) {
    if (!s || !out || layer < 0 || layer >= s->m->g.num_layers || len < 0 || len > s->max_ctx)
        return set_err(CASCADE_EINVAL, "bad arguments");
    const Dims D(s->m->g);
    CK(cudaSetDevice(s->m->device));
    CK(cudaStreamSynchronize(s->stream));
    const uint16_t* base = (which ? s->vc : s->kc) + (size_t)layer * D.KV * s->max_ctx * D.hd;
    for (int h = 0; h < D.KV; ++h)
        CK(cudaMemcpy(out + (size_t)h * len * D.hd, base + (size_t)h * s->max_ctx * D.hd, (size_t)len * D.hd * 2,
                      cudaMemcpyDeviceToHost));
    return CASCADE_OK;
}
