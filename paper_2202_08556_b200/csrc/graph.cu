// daspmm — DA-SpMM with on-device dispatch: select kernel -> SWITCH conditional node.
//
// One CUDA graph per (handle, model, operands, N, flags): node 0 is the selector
// kernel (select.cu), which computes the kernel id from the handle's device-resident
// features and calls cudaGraphSetConditional; node 1 is a SWITCH conditional with
// eight bodies, body k holding design-space kernel k (plus the EB prologue, plus a
// device transpose of B when kernel k needs the other layout, as spmm_auto_layout
// does, spmm.hpp:275-281). The host never learns the choice — no round trip — and a
// repeated call is a single cudaGraphLaunch.
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "dispatch.h"
#include "internal.h"

namespace daspmm {

namespace {

// Graph entries: the full operand key (the captured kernels bake in B, C and the stream).
struct Key {
    uint64_t model_gen;
    const void* B;
    int b_layout;
    int64_t ldb, N;
    void* C;
    int64_t ldc, W;
    unsigned flags;
    int64_t hw;
    cudaStream_t stream;
    bool operator==(const Key& o) const {
        return std::tie(model_gen, B, b_layout, ldb, N, C, ldc, W, flags, hw, stream) ==
               std::tie(o.model_gen, o.B, o.b_layout, o.ldb, o.N, o.C, o.ldc, o.W, o.flags, o.hw,
                        o.stream);
    }
};

// The selector's choice is a pure function of (matrix, model, N, hw) — operands never
// enter it — so once the device has published it, every later call with that key
// (any B, C, stream) launches the chosen kernel directly.
struct DecisionKey {
    uint64_t model_gen;
    int64_t N, hw;
    bool operator<(const DecisionKey& o) const {
        return std::tie(model_gen, N, hw) < std::tie(o.model_gen, o.N, o.hw);
    }
};

struct Entry {
    Key key{};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int* chunk_row = nullptr;
    void* bt = nullptr;       // B in the other layout (may be null: see twin fallback)
    int* own_kernel = nullptr;
    int* decision = nullptr;  // device cache of the selector's choice (-1 = not yet made)
    // The selector kernel also publishes its choice into mapped pinned host memory.
    int* published = nullptr;        // host view
    int* published_dev = nullptr;    // device view
    cudaEvent_t done = nullptr;      // recorded after the entry's last launch
    ~Entry() {
        // cudaGraphExecDestroy defers the release of an in-flight graph; the scratch
        // below is only freed once `done` has completed (retire / graph_cache_free).
        cudaFree(decision);
        if (published) cudaFreeHost(published);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        cudaFree(chunk_row);
        cudaFree(bt);
        cudaFree(own_kernel);
        if (done) cudaEventDestroy(done);
    }
    bool idle() const { return done == nullptr || cudaEventQuery(done) != cudaErrorNotReady; }
};

// At most kMaxGraphs instantiated graphs per handle (LRU); an evicted or decided entry is
// retired and freed once its last launch has completed.
constexpr size_t kMaxGraphs = 4;

struct Cache {
    std::mutex mu;
    std::map<DecisionKey, int> decided;
    std::list<std::unique_ptr<Entry>> lru;      // front = most recently used
    std::vector<std::unique_ptr<Entry>> retired;

    void reap() {
        for (size_t i = 0; i < retired.size();) {
            if (retired[i]->idle()) {
                retired[i] = std::move(retired.back());
                retired.pop_back();
            } else {
                ++i;
            }
        }
        cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
    }
    void retire(std::list<std::unique_ptr<Entry>>::iterator it) {
        retired.push_back(std::move(*it));
        lru.erase(it);
    }
    ~Cache() {
        for (auto& e : lru)
            if (e->done) cudaEventSynchronize(e->done);
        for (auto& e : retired)
            if (e->done) cudaEventSynchronize(e->done);
    }
};

int elem(int dtype) { return dtype == DASPMM_F64 ? 8 : 4; }

// Kernel ids 0..7 in pinned host memory: the direct path writes the caller's d_kernel
// with an async copy from here (a pageable source would serialise the stream).
const int* pinned_ids() {
    static int* ids = [] {
        int* p = nullptr;
        if (cudaHostAlloc(reinterpret_cast<void**>(&p), 8 * sizeof(int), cudaHostAllocDefault) !=
            cudaSuccess) {
            cudaGetLastError();
            static int fallback[8];
            p = fallback;
        }
        for (int i = 0; i < 8; ++i) p[i] = i;
        return p;
    }();
    return ids;
}

}  // namespace

void graph_cache_free(daspmm_csr* h) {
    delete static_cast<Cache*>(h->graph_cache);
    h->graph_cache = nullptr;
}

static int graph_cache_stats(const daspmm_csr* h, int64_t* graphs, int64_t* retired, int64_t* decided) {
    Cache* c = static_cast<Cache*>(h->graph_cache);
    int64_t g = 0, r = 0, d = 0;
    if (c) {
        std::lock_guard<std::mutex> lk(c->mu);
        c->reap();
        g = int64_t(c->lru.size());
        r = int64_t(c->retired.size());
        d = int64_t(c->decided.size());
    }
    if (graphs) *graphs = g;
    if (retired) *retired = r;
    if (decided) *decided = d;
    return DASPMM_OK;
}

static int build_entry(const daspmm_csr* h, const daspmm_model* m, const Key& k, bool reselect,
                       Entry& en) {
    cudaError_t e;
    en.key = k;
    if ((e = cudaMalloc(&en.own_kernel, sizeof(int))) != cudaSuccess)
        return cuda_fail(e, "graph: cudaMalloc");
    if ((e = cudaEventCreateWithFlags(&en.done, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "graph: event");
    if (int rc = ensure_coo(h, 0)) return rc;  // EB bodies read COO row ids
    if (!(k.flags & DASPMM_EXACT))
        if (int rc = ensure_tiles(h, 0)) return rc;  // RB+RM+SR body may walk the tiles
    // Scratch: EB chunk rows for the largest plan, and B in the other layout.
    int64_t max_p = 1;
    for (int kid = 4; kid < 8; ++kid) {
        const Plan p = plan_spmm(h, kid, 0, k.W, k.N, k.B, k.ldb, k.C, k.ldc,
                                 (k.flags & DASPMM_EXACT) != 0);
        max_p = std::max<int64_t>(max_p, p.P);
    }
    if ((e = cudaMalloc(&en.chunk_row, sizeof(int) * size_t(max_p))) != cudaSuccess)
        return cuda_fail(e, "graph: cudaMalloc(chunk_row)");
    // B in the other layout only when the caller asks for the reference's conversion;
    // otherwise a body whose kernel needs it runs the layout twin (below).
    const size_t bt_bytes = size_t(elem(h->dtype)) * size_t(h->K) * size_t(k.N);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    if ((k.flags & DASPMM_CONVERT_LAYOUT) && bt_bytes > 0 && bt_bytes <= free_b / 4) {
        if ((e = cudaMalloc(&en.bt, bt_bytes)) != cudaSuccess) en.bt = nullptr;
    }
    const int64_t ldt = k.b_layout == DASPMM_ROW_MAJOR ? std::max<int64_t>(h->K, 1)
                                                       : std::max<int64_t>(k.N, 1);

    if ((e = cudaMalloc(&en.decision, sizeof(int))) != cudaSuccess)
        return cuda_fail(e, "graph: cudaMalloc(decision)");
    if ((e = cudaMemset(en.decision, 0xff, sizeof(int))) != cudaSuccess)
        return cuda_fail(e, "graph: cudaMemset(decision)");
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&en.published), sizeof(int),
                           cudaHostAllocMapped)) != cudaSuccess)
        return cuda_fail(e, "graph: cudaHostAlloc(published)");
    *en.published = -1;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&en.published_dev), en.published,
                                      0)) != cudaSuccess)
        return cuda_fail(e, "graph: cudaHostGetDevicePointer");
    cudaStream_t cap;
    if ((e = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "graph: stream");
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{cap};

    if ((e = cudaGraphCreate(&en.graph, 0)) != cudaSuccess) return cuda_fail(e, "graph: create");
    cudaGraphConditionalHandle cond;
    if ((e = cudaGraphConditionalHandleCreate(&cond, en.graph, 8u, cudaGraphCondAssignDefault)) !=
        cudaSuccess)
        return cuda_fail(e, "graph: conditional handle");
    // Node 0: selector.
    if ((e = cudaStreamBeginCaptureToGraph(cap, en.graph, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
        return cuda_fail(e, "graph: capture(select)");
    // reselect (DASPMM_RESELECT): no device-side decision cache and no publication, so
    // every launch walks the ensemble and dispatches through the SWITCH node.
    int rc = launch_select(h, m, k.N, k.hw, en.own_kernel, cond, true, cap,
                           reselect ? nullptr : en.decision, reselect ? nullptr : en.published_dev);
    cudaGraph_t g_out = nullptr;
    e = cudaStreamEndCapture(cap, &g_out);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "graph: end capture(select)");
    size_t n_nodes = 0;
    cudaGraphGetNodes(en.graph, nullptr, &n_nodes);
    std::vector<cudaGraphNode_t> nodes(n_nodes);
    cudaGraphGetNodes(en.graph, nodes.data(), &n_nodes);
    // Node 1: SWITCH over the eight design-space kernels.
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeSwitch;
    cp.conditional.size = 8;
    cudaGraphNode_t sw;
    if ((e = cudaGraphAddNode(&sw, en.graph, nodes.data(), n_nodes, &cp)) != cudaSuccess)
        return cuda_fail(e, "graph: add switch node");
    for (int kid = 0; kid < 8; ++kid) {
        cudaGraph_t body = cp.conditional.phGraph_out[kid];
        const int want = ((kid >> 1) & 1) ? DASPMM_COL_MAJOR : DASPMM_ROW_MAJOR;
        int run_kid = kid;
        const void* Bk = k.B;
        int64_t ldk = k.ldb;
        bool need_t = want != k.b_layout;
        if (need_t && !en.bt) {
            run_kid = kid ^ 2;  // layout twin: same M/K choices, operand's layout
            need_t = false;
        }
        if ((e = cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0,
                                               cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
            return cuda_fail(e, "graph: capture(body)");
        if (need_t) {
            if (k.b_layout == DASPMM_ROW_MAJOR)
                e = transpose(h->dtype, k.B, h->K, k.N, k.ldb, en.bt, ldt, cap);
            else
                e = transpose(h->dtype, k.B, k.N, h->K, k.ldb, en.bt, ldt, cap);
            Bk = en.bt;
            ldk = ldt;
        }
        // make_config defaults (worker.hpp:47-55): W = 8 unless given.
        rc = e == cudaSuccess ? spmm_device(h, run_kid, 0, k.W, Bk, ldk, k.N, k.C, k.ldc,
                                            k.flags & DASPMM_EXACT, cap, en.chunk_row)
                              : cuda_fail(e, "graph: transpose");
        cudaGraph_t bo = nullptr;
        e = cudaStreamEndCapture(cap, &bo);
        if (rc) return rc;
        if (e != cudaSuccess) return cuda_fail(e, "graph: end capture(body)");
    }
    if ((e = cudaGraphInstantiate(&en.exec, en.graph, 0)) != cudaSuccess)
        return cuda_fail(e, "graph: instantiate");
    return DASPMM_OK;
}

}  // namespace daspmm

using namespace daspmm;

extern "C" int daspmm_spmm_selected(const daspmm_csr* h, const daspmm_model* m, int64_t hw,
                                    const void* d_B, int b_layout, int64_t ldb, int64_t N,
                                    void* d_C, int64_t ldc, int64_t W, unsigned flags,
                                    int* d_kernel, daspmm_stream stream) {
    if (!h || !m) return fail(DASPMM_ERR_INVALID_ARG, "spmm_selected: null argument");
    if (W <= 0) W = 8;
    const int want_kernel0 = b_layout == DASPMM_COL_MAJOR ? 2 : 0;
    if (int rc = check_call(h, want_kernel0, 0, W, 1, b_layout, ldb, N, ldc,
                            (flags & DASPMM_EXACT) != 0))
        return rc;
    if (h->M == 0)
        return fail(DASPMM_ERR_INVALID_ARG, "extract_features: matrix has no rows to summarize");
    int nc = 0, nf = 0, nr = 0, uh = 0;
    daspmm_model_info(m, &nc, &nf, &nr, &uh);
    if (uh && hw < 0)
        return fail(DASPMM_ERR_INVALID_ARG,
                    "encode_features: model expects a hardware_id but the sample has none");
    if (nf != (uh ? 5 : 4)) return fail(DASPMM_ERR_INVALID_ARG, "predict: feature count mismatch");
    // The SWITCH node has eight bodies; KernelId::from_index rejects any other class
    // (kernel_id.hpp:30), so a model that could predict one is refused up front.
    if (nc > 8) return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    if (N == 0) return DASPMM_OK;
    DeviceGuard g(h->device);
    daspmm_csr* hm = const_cast<daspmm_csr*>(h);
    {
        std::lock_guard<std::mutex> lk(hm->mu);
        if (!hm->graph_cache) hm->graph_cache = new Cache;
    }
    Cache* cache = static_cast<Cache*>(hm->graph_cache);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool reselect = (flags & DASPMM_RESELECT) != 0;
    const unsigned kflags = flags & ~unsigned(DASPMM_RESELECT);
    const DecisionKey dk{model_generation(m), N, uh ? hw : -1};
    // The key keeps the RESELECT bit: a reselect graph never publishes its choice, so a
    // plain call must not reuse it (it would never reach the direct steady state).
    const Key key{model_generation(m), d_B, b_layout, ldb, N, d_C, ldc, W, flags, uh ? hw : -1, s};

    int decided = -1;
    Entry* en = nullptr;
    {
        std::lock_guard<std::mutex> lk(cache->mu);
        // Entries whose selector has published: record the decision, retire the graph.
        for (auto it = cache->lru.begin(); it != cache->lru.end();) {
            const int pub = *reinterpret_cast<volatile int*>((*it)->published);
            if (pub >= 0 && pub < 8) {
                cache->decided[DecisionKey{(*it)->key.model_gen, (*it)->key.N, (*it)->key.hw}] = pub;
                auto nx = std::next(it);
                cache->retire(it);
                it = nx;
            } else {
                ++it;
            }
        }
        if (!reselect) {
            auto d = cache->decided.find(dk);
            if (d != cache->decided.end()) decided = d->second;
        }
        if (decided < 0) {
            for (auto it = cache->lru.begin(); it != cache->lru.end(); ++it) {
                if ((*it)->key == key) {
                    cache->lru.splice(cache->lru.begin(), cache->lru, it);
                    en = cache->lru.front().get();
                    break;
                }
            }
            if (!en) {
                // Freeing retired graphs synchronises (cudaFree, cudaFreeHost), so it is
                // done only here, on the already slow build path — never on a launch.
                cache->reap();
                auto fresh = std::make_unique<Entry>();
                if (int rc = build_entry(h, m, key, reselect, *fresh)) {
                    // A graph left mid-capture cannot be destroyed safely; leak it.
                    fresh->graph = nullptr;
                    return rc;
                }
                cache->lru.push_front(std::move(fresh));
                en = cache->lru.front().get();
                while (cache->lru.size() > kMaxGraphs) cache->retire(std::prev(cache->lru.end()));
            }
            cudaError_t e = cudaGraphLaunch(en->exec, s);
            if (e == cudaSuccess) e = cudaEventRecord(en->done, s);
            if (e == cudaSuccess && d_kernel)
                e = cudaMemcpyAsync(d_kernel, en->own_kernel, sizeof(int), cudaMemcpyDeviceToDevice, s);
            return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "graph launch");
        }
    }
    // Steady state: the device's published choice, launched directly. Scratch (EB chunk
    // rows, B in the other layout) is stream-ordered from the library pool.
    cudaError_t e = cudaSuccess;
    if (d_kernel)
        e = cudaMemcpyAsync(d_kernel, pinned_ids() + decided, sizeof(int), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "spmm_selected: kernel id");
    const int want = ((decided >> 1) & 1) ? DASPMM_COL_MAJOR : DASPMM_ROW_MAJOR;
    const unsigned xflags = kflags & DASPMM_EXACT;
    if (want == b_layout) return spmm_device(h, decided, 0, W, d_B, ldb, N, d_C, ldc, xflags, s, nullptr);
    if (!(kflags & DASPMM_CONVERT_LAYOUT))  // the layout twin on B as given
        return spmm_device(h, decided ^ 2, 0, W, d_B, ldb, N, d_C, ldc, xflags, s, nullptr);
    const size_t bytes = size_t(elem(h->dtype)) * size_t(h->K) * size_t(N);
    void* bt = nullptr;
    if (scratch_alloc(&bt, std::max<size_t>(bytes, 16), h->device, s) != cudaSuccess) {
        cudaGetLastError();  // no room for the other layout: the layout twin (same M/K choices)
        return spmm_device(h, decided ^ 2, 0, W, d_B, ldb, N, d_C, ldc, xflags, s, nullptr);
    }
    const int64_t ldt = b_layout == DASPMM_ROW_MAJOR ? std::max<int64_t>(h->K, 1)
                                                     : std::max<int64_t>(N, 1);
    e = b_layout == DASPMM_ROW_MAJOR ? transpose(h->dtype, d_B, h->K, N, ldb, bt, ldt, s)
                                     : transpose(h->dtype, d_B, N, h->K, ldb, bt, ldt, s);
    int rc = e == cudaSuccess ? spmm_device(h, decided, 0, W, bt, ldt, N, d_C, ldc, xflags, s, nullptr)
                              : cuda_fail(e, "transpose");
    scratch_free(bt, s);
    return rc;
}

extern "C" int daspmm_selected_cache_info(const daspmm_csr* h, int64_t* graphs, int64_t* retired,
                                          int64_t* decided) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "selected_cache_info: null handle");
    return graph_cache_stats(h, graphs, retired, decided);
}
