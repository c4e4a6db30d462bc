// daspmm — the data-aware selector (paper §5; selector.hpp, gbdt.hpp).
//
// Host side: parse the reference's selector text v1 (selector.hpp:113-132,
// gbdt.hpp:336-453) with the same validation and messages, keep the ensemble, and
// evaluate predict_kernel exactly as the reference (selector.hpp:62-65).
//
// Device side: the ensemble is flattened once. Every split is rewritten into an
// exact integer or interval test so the GPU decision cannot drift from the host's:
//   f0 = log2(max(nnz,1))  <= t   <=>  max(nnz,1)  <= icut  (icut found with the host's
//   f1 = log2(max(M,1))    <= t   <=>  max(M,1)    <= icut   own std::log2, so CUDA's
//                                                            log2 never enters)
//   f3 = (double)N         <= t   <=>  N   <= floor(t)
//   f4 = (double)hw        <= t   <=>  hw  <= floor(t)
//   f2 = std_row           <= t   decided from the handle's proven interval
//                                  [std_lo, std_hi]; if t falls inside it the kernel
//                                  replays the reference's sequential sum (cached).
// Per-class raw scores are then summed in round order with __dadd_rn and the argmax
// uses strict '>' (ties to the lowest class), as gbdt.hpp:60-77.
#include <cmath>
#include <cstring>
#include <atomic>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "exact_sum.cuh"
#include "internal.h"

namespace daspmm {

struct HostNode {
    int feature = -1;
    double threshold = 0.0;
    int left = -1, right = -1;
    double value = 0.0;
};

struct DevNode {
    int feature;  // -1 leaf
    int left;     // absolute node index
    int right;
    int pad;
    double thr;   // std_row threshold (feature 2)
    long long icut;  // integer cut for features 0, 1, 3, 4
    double value;
    double pad2;     // 48 bytes: runs of nodes are 16-B aligned for 1-D TMA staging
};
static_assert(sizeof(DevNode) == 48, "DevNode staged by cp.async.bulk in 16-B units");

}  // namespace daspmm

struct daspmm_model {
    uint64_t generation = 0;  // unique per parse; keys graph caches
    int num_classes = 0, num_features = 0, best_round = -1;
    bool uses_hardware = false;
    std::vector<std::vector<std::vector<daspmm::HostNode>>> rounds;  // [round][class]
    std::vector<int64_t> tree_off;                                  // flattened
    daspmm::DevNode* d_nodes = nullptr;
    int64_t* d_tree_off = nullptr;
    int64_t n_nodes = 0;
};

namespace daspmm {

namespace {

struct Parser {
    std::istringstream in;
    explicit Parser(std::string s) : in(std::move(s)) {}
    std::string err;
    template <class T>
    bool tok(T& v, const char* what) {
        if (!(in >> v)) {
            err = std::string("model stream truncated or malformed: expected ") + what;
            return false;
        }
        return true;
    }
    bool lit(const std::string& l) {
        std::string t;
        if (!tok(t, l.c_str())) return false;
        if (t != l) {
            err = "model stream malformed: expected '" + l + "', got '" + t + "'";
            return false;
        }
        return true;
    }
};

// Largest n >= 1 with std::log2((double)n) <= t, or 0 when none (t < 0).
long long log2_cut(double t) {
    if (!(std::log2(1.0) <= t)) return 0;
    long long lo = 1, hi = (1LL << 62);
    if (std::log2(double(hi)) <= t) return hi;
    while (hi - lo > 1) {
        const long long mid = lo + (hi - lo) / 2;
        if (std::log2(double(mid)) <= t) lo = mid;
        else hi = mid;
    }
    return lo;
}

long long floor_cut(double t) {
    if (t >= 9.0e18) return (1LL << 62);
    if (t < -9.0e18) return -(1LL << 62);
    return (long long)std::floor(t);
}

}  // namespace

int parse_model(const char* text, size_t len, daspmm_model** out) {
    Parser p(std::string(text, len));
    auto bad = [&](const std::string& m) { return fail(DASPMM_ERR_MODEL_FORMAT, m); };
    std::string tag, ver;
    if (!p.tok(tag, "selector tag") || !p.tok(ver, "selector version")) return bad(p.err);
    if (tag != "spmmkit-selector") return bad("not a selector stream (tag '" + tag + "')");
    if (ver != "v1") return bad("unsupported selector version '" + ver + "', expected v1");
    int uses_hw = 0;
    if (!p.lit("uses_hardware") || !p.tok(uses_hw, "uses_hardware flag")) return bad(p.err);
    if (!p.tok(tag, "format tag") || !p.tok(ver, "format version")) return bad(p.err);
    if (tag != "spmmkit-gbdt") return bad("not a model stream (tag '" + tag + "')");
    if (ver != "v1") return bad("unsupported model version '" + ver + "', expected v1");
    auto* m = new daspmm_model;
    static std::atomic<uint64_t> gen{1};
    m->generation = gen++;
    std::unique_ptr<daspmm_model> guard(m);
    m->uses_hardware = uses_hw != 0;
    if (!p.lit("classes") || !p.tok(m->num_classes, "class count") || !p.lit("features") ||
        !p.tok(m->num_features, "feature count") || !p.lit("best_round") ||
        !p.tok(m->best_round, "best round"))
        return bad(p.err);
    if (m->num_classes < 1 || m->num_features < 0) return bad("implausible class/feature counts");
    if (!p.lit("config")) return bad(p.err);
    {  // GbdtConfig fields with their reference types (gbdt.hpp:396-409)
        int iv;
        double dv;
        unsigned long long uv;
        if (!p.lit("num_rounds") || !p.tok(iv, "num_rounds") || !p.lit("max_depth") ||
            !p.tok(iv, "max_depth") || !p.lit("min_leaf") || !p.tok(iv, "min_leaf") ||
            !p.lit("learning_rate") || !p.tok(dv, "learning_rate") || !p.lit("patience") ||
            !p.tok(iv, "patience") || !p.lit("lambda") || !p.tok(dv, "lambda") ||
            !p.lit("seed") || !p.tok(uv, "seed"))
            return bad(p.err);
    }
    int n_names = 0;
    if (!p.lit("feature_names") || !p.tok(n_names, "feature name count")) return bad(p.err);
    if (n_names < 0 || n_names > 4096) return bad("implausible feature name count");
    for (int i = 0; i < n_names; ++i) {
        std::string nm;
        if (!p.tok(nm, "feature name")) return bad(p.err);
    }
    int n_rounds = 0;
    if (!p.lit("rounds") || !p.tok(n_rounds, "round count")) return bad(p.err);
    if (n_rounds < 0 || n_rounds > 1000000) return bad("implausible round count");
    m->rounds.resize(n_rounds);
    for (int r = 0; r < n_rounds; ++r) {
        m->rounds[r].resize(m->num_classes);
        for (int c = 0; c < m->num_classes; ++c) {
            int rr = 0, cc = 0, nn = 0;
            if (!p.lit("tree") || !p.tok(rr, "tree round") || !p.tok(cc, "tree class"))
                return bad(p.err);
            if (rr != r || cc != c) return bad("tree out of order");
            if (!p.tok(nn, "node count")) return bad(p.err);
            if (nn < 1 || nn > 10000000) return bad("implausible node count");
            auto& tree = m->rounds[r][c];
            tree.resize(nn);
            for (auto& nd : tree) {
                std::string kind;
                if (!p.lit("node") || !p.tok(kind, "node kind")) return bad(p.err);
                if (kind == "split") {
                    double gain;
                    if (!p.tok(nd.feature, "split feature") || !p.tok(nd.threshold, "split threshold") ||
                        !p.tok(nd.left, "left child") || !p.tok(nd.right, "right child") ||
                        !p.tok(gain, "split gain"))
                        return bad(p.err);
                    if (nd.feature >= m->num_features || nd.left < 0 || nd.right < 0 ||
                        nd.left >= nn || nd.right >= nn)
                        return bad("split node references out of range");
                } else if (kind == "leaf") {
                    nd.feature = -1;
                    if (!p.tok(nd.value, "leaf value")) return bad(p.err);
                } else {
                    return bad("unknown node kind '" + kind + "'");
                }
            }
        }
    }
    if (!p.lit("end")) return bad(p.err);

    // Flatten and upload.
    std::vector<DevNode> nodes;
    m->tree_off.push_back(0);
    for (int r = 0; r < n_rounds; ++r)
        for (int c = 0; c < m->num_classes; ++c) {
            const auto& tree = m->rounds[r][c];
            const int base = int(nodes.size());
            for (const auto& nd : tree) {
                DevNode d{};
                d.feature = nd.feature;
                d.left = nd.left >= 0 ? base + nd.left : -1;
                d.right = nd.right >= 0 ? base + nd.right : -1;
                d.thr = nd.threshold;
                d.value = nd.value;
                if (nd.feature == 0 || nd.feature == 1) d.icut = log2_cut(nd.threshold);
                else if (nd.feature >= 3) d.icut = floor_cut(nd.threshold);
                nodes.push_back(d);
            }
            m->tree_off.push_back(int64_t(nodes.size()));
        }
    m->n_nodes = int64_t(nodes.size());
    if (daspmm_device_count() > 0 && !nodes.empty()) {
        cudaError_t e;
        if ((e = cudaMalloc(&m->d_nodes, sizeof(DevNode) * nodes.size())) != cudaSuccess ||
            (e = cudaMalloc(&m->d_tree_off, sizeof(int64_t) * m->tree_off.size())) != cudaSuccess)
            return cuda_fail(e, "model upload");
        if ((e = cudaMemcpy(m->d_nodes, nodes.data(), sizeof(DevNode) * nodes.size(),
                            cudaMemcpyHostToDevice)) != cudaSuccess ||
            (e = cudaMemcpy(m->d_tree_off, m->tree_off.data(),
                            sizeof(int64_t) * m->tree_off.size(), cudaMemcpyHostToDevice)) !=
                cudaSuccess)
            return cuda_fail(e, "model upload");
    }
    *out = guard.release();
    return DASPMM_OK;
}

// encode_features (selector.hpp:19-33) + predict_class (gbdt.hpp:60-77) on the host.
int predict_host(const daspmm_model* m, int64_t nnz, int64_t mat_size, double std_row,
                 int64_t n_cols, int64_t hw, int* kernel) {
    std::vector<double> f{std::log2(double(std::max<int64_t>(nnz, 1))),
                          std::log2(double(std::max<int64_t>(mat_size, 1))), std_row,
                          double(n_cols)};
    if (m->uses_hardware) {
        if (hw < 0)
            return fail(DASPMM_ERR_INVALID_ARG,
                        "encode_features: model expects a hardware_id but the sample has none");
        f.push_back(double(hw));
    }
    if (int(f.size()) != m->num_features)
        return fail(DASPMM_ERR_INVALID_ARG, "predict: got " + std::to_string(f.size()) +
                                                " features, model expects " +
                                                std::to_string(m->num_features));
    std::vector<double> s(m->num_classes, 0.0);
    for (const auto& round : m->rounds)
        for (int c = 0; c < m->num_classes; ++c) {
            const auto& t = round[c];
            int i = 0;
            while (t[i].feature >= 0) i = f[t[i].feature] <= t[i].threshold ? t[i].left : t[i].right;
            s[c] += t[i].value;
        }
    int best = 0;
    for (int c = 1; c < m->num_classes; ++c)
        if (s[c] > s[best]) best = c;
    if (best < 0 || best > 7) return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    *kernel = best;
    return DASPMM_OK;
}

// ------------------------------------------------------------------ device selector
constexpr int kSelThreads = 256;
constexpr int kMaxClasses = 16;

// Decision for one split; returns 0/1, or 2 when the std interval is ambiguous.
__device__ __forceinline__ int decide(const DevNode& nd, long long f0, long long f1, long long f3,
                                      long long f4, double std_lo, double std_hi, bool have_exact,
                                      double std_exact) {
    switch (nd.feature) {
        case 0: return f0 <= nd.icut;
        case 1: return f1 <= nd.icut;
        case 3: return f3 <= nd.icut;
        case 4: return f4 <= nd.icut;
        default:
            if (have_exact) return std_exact <= nd.thr;
            if (nd.thr < std_lo) return 0;
            if (nd.thr >= std_hi) return 1;
            return 2;
    }
}

__global__ void __launch_bounds__(kSelThreads)
k_select(const DevNode* __restrict__ nodes, const int64_t* __restrict__ tree_off, int num_rounds,
         int num_classes, const int* __restrict__ rp, DevFeatures* feat, long long n_cols,
         long long hw, int* out_kernel, cudaGraphConditionalHandle cond, int use_cond,
         int* cache, volatile int* publish) {
    extern __shared__ double leaf[];  // [num_rounds * num_classes]
    // The decision is a pure function of (matrix, model, N, hw): a graph that already
    // made it re-applies it without walking the ensemble again.
    if (cache != nullptr) {
        const int cached = *cache;
        if (cached >= 0) {
            if (threadIdx.x == 0) {
                *out_kernel = cached;
                if (publish != nullptr) *publish = cached;
                if (use_cond) cudaGraphSetConditional(cond, unsigned(cached));
            }
            return;
        }
    }
    __shared__ int ambiguous;
    __shared__ double s_exact;
    __shared__ int s_have;
    __shared__ double scores[kMaxClasses];
    if (threadIdx.x == 0) {
        ambiguous = 0;
        s_have = feat->exact_valid;
        s_exact = feat->std_exact;
    }
    __syncthreads();
    const long long nnz = feat->nnz > 1 ? feat->nnz : 1;
    const long long rows = feat->rows > 1 ? feat->rows : 1;
    const double lo = feat->std_lo, hi = feat->std_hi;
    const int ntrees = num_rounds * num_classes;
    for (int pass = 0; pass < 2; ++pass) {
        const bool have = s_have != 0;
        const double ex = s_exact;
        for (int t = threadIdx.x; t < ntrees; t += kSelThreads) {
            int i = int(tree_off[t]);
            bool amb = false;
            while (true) {
                const DevNode nd = nodes[i];
                if (nd.feature < 0) break;
                const int d = decide(nd, nnz, rows, n_cols, hw, lo, hi, have, ex);
                if (d == 2) {
                    amb = true;
                    break;
                }
                i = d ? nd.left : nd.right;
            }
            if (amb) atomicOr(&ambiguous, 1);
            else leaf[t] = nodes[i].value;
        }
        __syncthreads();
        if (!ambiguous) break;
        // Rare: a std_row threshold inside the proven interval. Replay the
        // reference's sequential sum once (features.hpp:27-35, the block-wide exact sum
        // of exact_sum.cuh) and cache it.
        {
            const int M = int(feat->rows);
            const double ss = M > 0 ? exact_sequential_sum<kSelThreads>(rp, M, feat->mean) : 0.0;
            if (threadIdx.x == 0) {
                const double sd = M > 0 ? __dsqrt_rn(__ddiv_rn(ss, double(M))) : 0.0;
                feat->std_exact = sd;
                feat->exact_valid = 1;
                s_exact = sd;
                s_have = 1;
                ambiguous = 0;
            }
        }
        __syncthreads();
    }
    // raw_scores: per class, sum over rounds in order from 0.0 (gbdt.hpp:60-65).
    if (threadIdx.x < num_classes) {
        double s = 0.0;
        for (int r = 0; r < num_rounds; ++r) s = __dadd_rn(s, leaf[r * num_classes + threadIdx.x]);
        scores[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int c = 1; c < num_classes; ++c)
            if (scores[c] > scores[best]) best = c;
        *out_kernel = best;
        if (cache != nullptr) *cache = best;
        if (publish != nullptr) *publish = best;  // mapped pinned host memory
        if (use_cond) cudaGraphSetConditional(cond, unsigned(best));
    }
}

// The same decision from a cluster of kSelCta CTAs: CTA q stages the nodes of its
// contiguous run of trees into shared memory with coalesced 16-byte loads (one pass over
// the model instead of a chain of dependent global loads per tree level), each thread
// walks one tree there, and CTA 0 gathers the leaves through distributed shared memory
// and sums them per class in round order (gbdt.hpp:60-65). Bits are those of k_select.
// A std_row split inside the proven interval sends CTA 0 down k_select's path (exact
// replay, then every tree walked again from global memory).
constexpr int kSelCta = 8;
struct SelRuns {  // node run [n[q], n[q+1]) of CTA q, from the host's tree offsets
    long long n[kSelCta + 1];
};

__global__ void __cluster_dims__(kSelCta, 1, 1) __launch_bounds__(kSelThreads)
k_select_cluster(const DevNode* __restrict__ nodes, const int64_t* __restrict__ tree_off,
                 int num_rounds, int num_classes, int per_cta, int stage_nodes, SelRuns runs,
                 const int* __restrict__ rp, DevFeatures* feat, long long n_cols, long long hw,
                 int* out_kernel, cudaGraphConditionalHandle cond, int use_cond, int* cache,
                 volatile int* publish) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned q = cluster.block_rank();
    if (cache != nullptr) {  // every CTA reads the same value: only CTA 0 writes it, last
        const int cached = *cache;
        if (cached >= 0) {
            if (q == 0 && threadIdx.x == 0) {
                *out_kernel = cached;
                if (publish != nullptr) *publish = cached;
                if (use_cond) cudaGraphSetConditional(cond, unsigned(cached));
            }
            return;
        }
    }
    extern __shared__ __align__(16) unsigned char sel_smem[];  // TMA destination: 16-B aligned
    // [stage_nodes DevNode][per_cta doubles: this CTA's leaves][ntrees doubles: CTA 0's]
    DevNode* snodes = reinterpret_cast<DevNode*>(sel_smem);
    double* my_leaf = reinterpret_cast<double*>(snodes + stage_nodes);
    double* all_leaf = my_leaf + per_cta;
    __shared__ int amb;
    __shared__ int any_amb;
    __shared__ double scores[kMaxClasses];
    const int ntrees = num_rounds * num_classes;
    const int t0 = min(int(q) * per_cta, ntrees), t1 = min(t0 + per_cta, ntrees);
    const int64_t n0 = runs.n[q], n1 = runs.n[q + 1];
    const bool staged = n1 - n0 <= stage_nodes;
    if (threadIdx.x == 0) amb = 0;
    __shared__ __align__(8) uint64_t bar;
    // One 1-D TMA bulk copy of the CTA's node run (one elected thread, mbarrier
    // completion); the first tree's root offset is loaded while it is in flight.
    const unsigned bytes = unsigned(n1 - n0) * unsigned(sizeof(DevNode));
    if (staged && threadIdx.x == 0) mbar_init(&bar, 1);
    __syncthreads();
    if (staged && threadIdx.x == 0 && bytes > 0) {
        mbar_expect_tx(&bar, bytes);
        bulk_g2s(snodes, nodes + n0, bytes, &bar);
    }
    const int64_t root0 = t0 + int(threadIdx.x) < t1 ? __ldg(tree_off + t0 + threadIdx.x) : 0;
    const long long nnz = feat->nnz > 1 ? feat->nnz : 1;
    const long long rows = feat->rows > 1 ? feat->rows : 1;
    const double lo = feat->std_lo, hi = feat->std_hi;
    const bool have = feat->exact_valid != 0;
    const double ex = feat->std_exact;
    if (staged && bytes > 0) mbar_wait(&bar, 0);
    for (int t = t0 + int(threadIdx.x); t < t1; t += blockDim.x) {
        int64_t i = t == t0 + int(threadIdx.x) ? root0 : tree_off[t];  // absolute index
        bool ambiguous = false;
        while (true) {
            const DevNode nd = staged ? snodes[i - n0] : nodes[i];
            if (nd.feature < 0) break;
            const int d = decide(nd, nnz, rows, n_cols, hw, lo, hi, have, ex);
            if (d == 2) {
                ambiguous = true;
                break;
            }
            i = d ? nd.left : nd.right;
        }
        if (ambiguous) amb = 1;
        else my_leaf[t - t0] = staged ? snodes[i - n0].value : nodes[i].value;
    }
    cluster.sync();  // every CTA's leaves and flag are in its shared memory
    if (q == 0) {
        if (threadIdx.x == 0) {
            int a = 0;
            for (unsigned r = 0; r < unsigned(kSelCta); ++r) a |= *cluster.map_shared_rank(&amb, r);
            any_amb = a;
        }
        __syncthreads();
        if (!any_amb) {
            for (int t = threadIdx.x; t < ntrees; t += blockDim.x) {
                const int r = t / per_cta;
                all_leaf[t] = cluster.map_shared_rank(my_leaf, unsigned(r))[t - r * per_cta];
            }
        }
    }
    cluster.sync();  // the peers' shared memory may go away after this
    if (q != 0) return;
    if (any_amb) {
        // Rare: replay the reference's sequential std_row sum (features.hpp:27-35) once,
        // cache it, and walk every tree again with the exact value.
        const int M = int(feat->rows);
        const double ss = M > 0 ? exact_sequential_sum<kSelThreads>(rp, M, feat->mean) : 0.0;
        const double sd = M > 0 ? __dsqrt_rn(__ddiv_rn(ss, double(M))) : 0.0;
        if (threadIdx.x == 0) {
            feat->std_exact = sd;
            feat->exact_valid = 1;
        }
        for (int t = threadIdx.x; t < ntrees; t += blockDim.x) {
            int64_t i = tree_off[t];
            while (true) {
                const DevNode nd = nodes[i];
                if (nd.feature < 0) break;
                i = decide(nd, nnz, rows, n_cols, hw, lo, hi, true, sd) ? nd.left : nd.right;
            }
            all_leaf[t] = nodes[i].value;
        }
        __syncthreads();
    }
    if (threadIdx.x < num_classes) {
        double s = 0.0;
#pragma unroll 10
        for (int r = 0; r < num_rounds; ++r) s = __dadd_rn(s, all_leaf[r * num_classes + threadIdx.x]);
        scores[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = 0;
        for (int c = 1; c < num_classes; ++c)
            if (scores[c] > scores[best]) best = c;
        *out_kernel = best;
        if (cache != nullptr) *cache = best;
        if (publish != nullptr) *publish = best;
        if (use_cond) cudaGraphSetConditional(cond, unsigned(best));
    }
}

uint64_t model_generation(const daspmm_model* m) { return m->generation; }

int launch_select(const daspmm_csr* h, const daspmm_model* m, int64_t n_cols, int64_t hw,
                  int* d_kernel, cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t s,
                  int* cache, int* publish) {
    const int ntrees = int(m->rounds.size()) * m->num_classes;
    if (m->num_classes > kMaxClasses)
        return fail(DASPMM_ERR_UNSUPPORTED, "select: more than 16 classes");
    // Cluster path: the largest per-CTA node run staged in shared memory (~100 KB for
    // the shipped 100-round, depth-4, 8-class model); beyond 200 KB the CTAs walk their
    // trees in global memory. DASPMM_SELECT_ONE_CTA=1 keeps the one-CTA kernel.
    static const bool one_cta = [] {
        const char* v = std::getenv("DASPMM_SELECT_ONE_CTA");
        return v && v[0] == '1';
    }();
    if (!one_cta && ntrees >= kSelCta) {
        const int per_cta = (ntrees + kSelCta - 1) / kSelCta;
        int64_t most = 0;
        SelRuns runs{};
        for (int q = 0; q <= kSelCta; ++q)
            runs.n[q] = m->tree_off[size_t(std::min(q * per_cta, ntrees))];
        for (int q = 0; q < kSelCta; ++q) most = std::max<int64_t>(most, runs.n[q + 1] - runs.n[q]);
        const size_t leaves = sizeof(double) * size_t(per_cta + ntrees);
        int stage = int(most);
        if (sizeof(DevNode) * size_t(stage) + leaves > 200 * 1024) stage = 0;
        const size_t smem = sizeof(DevNode) * size_t(stage) + leaves;
        if (smem <= 200 * 1024) {
            if (smem > 48 * 1024)
                cudaFuncSetAttribute(k_select_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem));
            k_select_cluster<<<kSelCta, kSelThreads, smem, s>>>(
                m->d_nodes, m->d_tree_off, int(m->rounds.size()), m->num_classes, per_cta, stage,
                runs, h->rp, h->d_feat, n_cols, hw, d_kernel, cond, use_cond ? 1 : 0, cache, publish);
            cudaError_t e = cudaGetLastError();
            return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "select");
        }
    }
    const size_t smem = sizeof(double) * size_t(std::max(ntrees, 1));
    if (smem > 200 * 1024) return fail(DASPMM_ERR_UNSUPPORTED, "select: ensemble too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k_select<<<1, kSelThreads, smem, s>>>(m->d_nodes, m->d_tree_off, int(m->rounds.size()),
                                          m->num_classes, h->rp, h->d_feat, n_cols, hw, d_kernel,
                                          cond, use_cond ? 1 : 0, cache, publish);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "select");
}

}  // namespace daspmm

using namespace daspmm;

extern "C" {

int daspmm_model_parse(const char* text, size_t len, daspmm_model** out) {
    if (!text || !out) return fail(DASPMM_ERR_INVALID_ARG, "model_parse: null argument");
    *out = nullptr;
    return parse_model(text, len, out);
}

int daspmm_model_destroy(daspmm_model* m) {
    if (!m) return DASPMM_OK;
    cudaFree(m->d_nodes);
    cudaFree(m->d_tree_off);
    delete m;
    return DASPMM_OK;
}

int daspmm_model_info(const daspmm_model* m, int* nc, int* nf, int* nr, int* uh) {
    if (!m) return fail(DASPMM_ERR_INVALID_ARG, "model_info: null model");
    if (nc) *nc = m->num_classes;
    if (nf) *nf = m->num_features;
    if (nr) *nr = int(m->rounds.size());
    if (uh) *uh = m->uses_hardware ? 1 : 0;
    return DASPMM_OK;
}

int daspmm_model_predict_host(const daspmm_model* m, int64_t nnz, int64_t mat_size, double std_row,
                              int64_t n_cols, int64_t hw, int* kernel) {
    if (!m || !kernel) return fail(DASPMM_ERR_INVALID_ARG, "predict: null argument");
    return predict_host(m, nnz, mat_size, std_row, n_cols, hw, kernel);
}

int daspmm_select(const daspmm_csr* h, const daspmm_model* m, int64_t n_cols, int64_t hw,
                  int* d_kernel, daspmm_stream stream) {
    if (!h || !m || !d_kernel) return fail(DASPMM_ERR_INVALID_ARG, "select: null argument");
    if (m->uses_hardware && hw < 0)
        return fail(DASPMM_ERR_INVALID_ARG,
                    "encode_features: model expects a hardware_id but the sample has none");
    if (m->num_features != (m->uses_hardware ? 5 : 4))
        return fail(DASPMM_ERR_INVALID_ARG, "predict: feature count mismatch");
    if (h->M == 0)
        return fail(DASPMM_ERR_INVALID_ARG, "extract_features: matrix has no rows to summarize");
    if (m->num_classes > 8) return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    if (!m->d_nodes) return fail(DASPMM_ERR_CUDA, "select: model not resident on a device");
    DeviceGuard g(h->device);
    return launch_select(h, m, n_cols, hw, d_kernel, cudaGraphConditionalHandle{}, false,
                         static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

}  // extern "C"
