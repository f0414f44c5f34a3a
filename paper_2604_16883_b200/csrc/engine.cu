// engine.cu — host side of the B200 SinkRouter engine and its C-ABI
// (include/sinkr_cuda.h).  Owns the HBM-resident KV cache, the anchor table,
// the per-step work buffers, the TMA tensor maps and one CUDA graph per
// (queries, outputs, mode) binding that replays probe -> decode -> combine.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <new>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/sinkr_cuda.h"
#include "host_util.hpp"
#include "step.cuh"
#include "analysis.cuh"
#include "span.hpp"

namespace {

using namespace sinkr;
using sinkr::host::Error;
using sinkr::host::fail;
using sinkr::host::g_err;
using sinkr::host::guard;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess)                                                         \
            fail(SINKR_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

// f32 -> bf16 round-to-nearest-even (bit-identical to __float2bfloat16_rn for
// finite inputs and to oracle/sinkr_oracle.c:orc_round_bf16).
uint16_t f32_to_bf16(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    if ((b & 0x7F800000u) == 0x7F800000u) return (uint16_t)((b >> 16) | ((x != x) ? 0x40u : 0u));
    return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}
float bf16_to_f32(uint16_t h) {
    const uint32_t b = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// router.cpp:59-65 with the reference's expression order.  Compiled for the
// host without FMA contraction (see build flags), like the reference.
double threshold_for_length(size_t len, const sinkr_threshold_profile& p) {
    if (len == 0) fail(SINKR_INVALID_ARGUMENT, "context length must be positive");
    const double x = static_cast<double>(len) / p.length_normalizer;
    const double tau = ((p.coeffs[0] * x + p.coeffs[1]) * x + p.coeffs[2]) * x + p.coeffs[3];
    return tau < p.clamp_lo ? p.clamp_lo : (p.clamp_hi < tau ? p.clamp_hi : tau);
}

bool layer_excluded(size_t layer, const sinkr_routing_config& c) {
    for (size_t i = 0; i < c.num_excluded_layers; ++i)
        if (c.excluded_layers[i] == layer) return true;
    return false;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            fail(SINKR_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int D>
int smem_bytes() {
    return dev::Cfg<D>::kSmemBytes;
}

}  // namespace

// Static share (percent of a CTA's fair share of the Active tokens) of the
// step kernel's unit-affine schedule; SINKR_STATIC_PCT overrides (A/B runs).
// 20 %: L2-flushed 512K routed 129.5-130.0 -> 127.0 us, back to back
// +0.4 us, 32K / 64K neutral (profiles/r02_static_ab.txt).
static uint32_t static_pct() {
    static uint32_t v = [] {
        const char* s = std::getenv("SINKR_STATIC_PCT");
        return s ? (uint32_t)std::atoi(s) : 20u;
    }();
    return v;
}
// Stages of its first static range a CTA prefetches into L2 under the layer's
// previous Active set (StepTables.spec_stages); SINKR_SPEC_STAGES overrides.
static uint32_t spec_stages() {
    static uint32_t v = [] {
        const char* s = std::getenv("SINKR_SPEC_STAGES");
        return s ? (uint32_t)std::atoi(s) : 8u;
    }();
    return v;
}
// Code prewarm of the single-sequence step (StepTables.prewarm: region bit
// mask, 8 = all regions in CTA G-1); SINKR_PREWARM overrides (A/B runs).
static uint32_t prewarm_default() {
    static uint32_t v = [] {
        const char* s = std::getenv("SINKR_PREWARM");
        return s ? (uint32_t)std::atoi(s) : 8u;
    }();
    return v;
}

struct sinkr_engine {
    sinkr_cache_config cfg{};
    size_t B = 1, U = 0, r = 0, D = 0, layers = 0, cap = 0;
    int device = 0, num_sms = 0, grid = 0, probe_grid = 1;
    uint32_t* d_head_degen = nullptr;
    cudaStream_t stream = nullptr;

    __nv_bfloat16* d_k = nullptr;
    __nv_bfloat16* d_v = nullptr;
    float* d_anchor = nullptr;
    float* d_anchor_norm = nullptr;
    double* d_norm64 = nullptr;
    std::vector<size_t> len;  // [layers][B][Hkv]
    std::vector<float> h_anchor, h_anchor_norm;
    std::vector<uint8_t> anchored;

    // step input block: hdr | tau[B] | len[B] | q[B][Hq][D] | k_new, v_new [B][Hkv][D]
    // (the new-token rows only travel with sinkr_decode_append_step)
    size_t off_tau = 0, off_len = 0, off_q = 0, in_bytes = 0;
    size_t off_kvn = 0, in_bytes_append = 0;
    // device copy of the slot lengths, advanced by append_token_kernel; the
    // host paths mark it stale and the next token append re-uploads it
    uint32_t* d_len = nullptr;
    uint32_t* h_len_stage = nullptr;  // pinned
    bool dlen_dirty = true;
    uint8_t* d_in = nullptr;
    uint8_t* h_in = nullptr;
    // step result block: out | head_scores | group_scores | tokens | flags
    size_t off_hs = 0, off_gs = 0, off_tok = 0, off_fl = 0, off_status = 0, res_bytes = 0;
    uint8_t* d_res = nullptr;
    uint8_t* h_res = nullptr;      // pinned + mapped
    uint8_t* h_res_dev = nullptr;  // device address of h_res (zero-copy results)
    uint8_t* h_in_dev = nullptr;   // device address of h_in (read by the upload kernel)
    // completion word of a host-buffer step (pinned + mapped): the host
    // clears it, the step kernel's last CTA sets it after a system fence, and
    // the blocking call spins on it instead of synchronising the stream
    uint32_t* h_done = nullptr;
    uint32_t* h_done_dev = nullptr;
    uint8_t* d_score_scratch = nullptr;  // sinkr_collect_scores_batch (grown on demand)
    size_t score_scratch_bytes = 0;

    dev::WorkState* d_ws = nullptr;
    uint32_t* d_active = nullptr;
    uint32_t* d_prefix = nullptr;
    uint32_t* d_slot_count = nullptr;
    float* d_partials = nullptr;
    size_t S = 0, PS = 0;
    // fused single-kernel step (step.cuh); the 3-kernel pipeline remains for
    // A/B profiling (SINKR_FUSED=0) and serves the multi-rank merge.
    bool fused = true;
    bool lean = false;  // single-sequence step-kernel instantiation (step.cuh LEAN)
    bool wide = false;  // GQA width 9-16: the step kernel's WIDE form (two 8-head tiles)
    dev::StepState* d_ss = nullptr;
    uint32_t* d_cursor = nullptr;
    uint32_t* d_tokens_done = nullptr;
    uint32_t* d_route_flags = nullptr;  // distributed routing decisions [U]
    uint8_t* d_span = nullptr;           // attend_chunk over a cached range: q | partial | scratch
    size_t span_bytes = 0;
    uint8_t* d_bos = nullptr;            // analysis scratch (run_bos), grown on demand
    size_t bos_bytes = 0;
    uint8_t* h_bos = nullptr;            // pinned + mapped staging for run_bos (prefix up, alpha0 down)
    uint8_t* h_bos_dev = nullptr;        // device address of h_bos
    cudaEvent_t ev_bos[2] = {};          // around run_bos's kernels (device time)
    // run_bos as captured graphs, keyed by (layer, u_first, n_units, G, weights,
    // parity, T); dropped when the scratch or the pinned staging is reallocated
    std::map<std::array<uint64_t, 7>, cudaGraphExec_t> bos_graphs;
    void drop_bos_graphs() {
        for (auto& kv : bos_graphs) cudaGraphExecDestroy(kv.second);
        bos_graphs.clear();
    }
    uint32_t bos_parity = 0;             // which counter set the next run_bos uses
    float bos_ms = -1.f;
    size_t h_bos_bytes = 0;
    uint32_t* d_ovf = nullptr;          // spill-slot lock + valid per unit [2][U]
    uint32_t* d_route_sum = nullptr;    // [grid] per-CTA Active bitmasks (distributed routing)
    uint32_t* d_spec_mask = nullptr;    // [layers] Active bitmask of each layer's last single-sequence step
    uint32_t* d_cta_epoch = nullptr;    // [2][grid]: step-kernel launches, mode-3 steps per CTA slot
    unsigned long long* d_trace = nullptr;  // SINKR_TRACE=1: per-CTA phase stamps
    // sequence-sharded peer merge (mode 3): this rank's exchange block
    // [2][world][U][PS] LL words {f32, step tag}, and every rank's block mapped here
    uint8_t* d_xchg = nullptr;
    size_t xchg_words = 0, xchg_bytes = 0;
    uint32_t world = 0, rank = 0;
    unsigned long long** d_peer_xchg = nullptr;  // device array [world]: every rank's exchange block
    std::vector<void*> ipc_opened;           // peer blocks opened through CUDA IPC
    // a peer-merge watchdog timeout leaves the ranks' step tags out of step
    // (the late rank still counts the step it never finished): the exchange
    // is unusable until every rank sets it up again
    bool peer_poisoned = false;

    CUtensorMap tmk{}, tmv{};
    CUtensorMap* d_tmap = nullptr;  // device copies of tmk, tmv (fused kernel)
    cudaEvent_t ev[4] = {};
    cudaEvent_t ev_in = nullptr;
    bool ev_in_pending = false;  // ev_in recorded since the last wait (else a wait is a no-op API call)
    bool timing = true;
    bool step_events = false;  // events around graph replays (last_step_stats step_ms)
    bool params_valid = false;
    std::vector<uint8_t> last_params;
    struct GraphEntry {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t probe = nullptr;  // the node whose ProbeParams are patched
        cudaKernelNodeParams probe_kp{};
        dev::DevTables probe_t{};
        dev::StepTables step_t{};
        bool fused = false;
        dev::ProbeParams pp{};
    };
    std::map<std::tuple<const void*, void*, int>, GraphEntry> graphs;
    dev::ProbeParams pp{};  // this step's probe parameters (staged by stage_params)
    uint32_t last_launches = 0;
    int last_mode = 0;

    size_t slot_index(size_t layer, size_t seq, size_t g) const {
        return (layer * B + seq) * cfg.num_kv_heads + g;
    }
    size_t row_base(size_t layer, size_t seq, size_t g) const {
        return slot_index(layer, seq, g) * cap;
    }
    dev::DevTables tables(const float* q) const {
        dev::DevTables t{};
        t.hdr = reinterpret_cast<const dev::StepHdr*>(d_in);
        t.tau = reinterpret_cast<const double*>(d_in + off_tau);
        t.len = reinterpret_cast<const uint32_t*>(d_in + off_len);
        t.q = q;
        t.anchors = d_anchor;
        t.anchor_norm = d_anchor_norm;
        t.head_scores = reinterpret_cast<double*>(d_res + off_hs);
        t.head_degen = d_head_degen;
        t.group_scores = reinterpret_cast<double*>(d_res + off_gs);
        t.unit_flags = reinterpret_cast<uint32_t*>(d_res + off_fl);
        t.tokens = reinterpret_cast<unsigned long long*>(d_res + off_tok);
        t.ws = d_ws;
        t.act_info = reinterpret_cast<uint4*>(d_active);
        t.unit_next = d_prefix;
        t.slot_count = d_slot_count;
        t.partials = d_partials;
        t.B = (uint32_t)B;
        t.Hq = (uint32_t)cfg.num_q_heads;
        t.Hkv = (uint32_t)cfg.num_kv_heads;
        t.r = (uint32_t)r;
        t.D = (uint32_t)D;
        t.cap = (uint32_t)cap;
        t.S = (uint32_t)S;
        t.grid = (uint32_t)grid;
        t.qscale = (1.0f / std::sqrt((float)D)) * 1.4426950408889634f;
        return t;
    }
    dev::StepTables step_tables(const float* q, float* out, int mode,
                                uint8_t* res = nullptr) const {
        if (!res) res = d_res;
        dev::StepTables t{};
        t.tmk = d_tmap;
        t.tmv = d_tmap + 1;
        t.q = q;
        t.anchors = d_anchor;
        t.anchor_norm = d_anchor_norm;
        t.tau_g = reinterpret_cast<const double*>(d_in + off_tau);
        t.len_g = reinterpret_cast<const uint32_t*>(d_in + off_len);
        t.head_scores = reinterpret_cast<double*>(res + off_hs);
        t.group_scores = reinterpret_cast<double*>(res + off_gs);
        t.unit_flags = reinterpret_cast<uint32_t*>(res + off_fl);
        t.tokens = reinterpret_cast<unsigned long long*>(res + off_tok);
        t.status = reinterpret_cast<uint32_t*>(res + off_status);
        t.ss = d_ss;
        t.cursor = d_cursor;
        t.slot_count = d_slot_count;
        t.tokens_done = d_tokens_done;
        t.route_flags = d_route_flags;
        t.route_sum = d_route_sum;
        t.ovf = d_ovf;
        t.cta_epoch = d_cta_epoch;
        t.partials = d_partials;
        t.out = out;
        t.B = (uint32_t)B;
        t.Hq = (uint32_t)cfg.num_q_heads;
        t.Hkv = (uint32_t)cfg.num_kv_heads;
        t.r = (uint32_t)r;
        t.cap = (uint32_t)cap;
        t.S = (uint32_t)S;
        t.mode = (uint32_t)mode;
        t.qscale = (1.0f / std::sqrt((float)D)) * 1.4426950408889634f;
        t.static_pct = static_pct();
        t.prewarm = prewarm_default();
        t.spec_mask = d_spec_mask;
        t.spec_stages = spec_stages();
        t.trace = d_trace;
        if (mode == 3) {
            t.peer_xchg = d_peer_xchg;
            t.xchg_local = reinterpret_cast<const unsigned long long*>(d_xchg);
            t.world = world;
            t.rank = rank;
        }
        return t;
    }
    uint32_t* clocks() const { return reinterpret_cast<uint32_t*>(d_res + off_status) + 4; }
};

namespace {

void check_slot(const sinkr_engine* e, size_t seq, size_t layer, size_t kv_head) {
    if (layer >= e->layers) fail(SINKR_OUT_OF_RANGE, "layer index out of range");
    if (kv_head >= e->cfg.num_kv_heads) fail(SINKR_OUT_OF_RANGE, "kv_head index out of range");
    if (seq >= e->B) fail(SINKR_OUT_OF_RANGE, "sequence index out of range");
}

void make_tmap(CUtensorMap* map, void* base, size_t rows, size_t D) {
    const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(D * 2)};
    const cuuint32_t box[2] = {(cuuint32_t)(D >= 64 ? 64 : D), (cuuint32_t)dev::kStageTok};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw =
        D >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    const CUresult rc = get_encode()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides,
                                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) fail(SINKR_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
}

int probe_smem(const sinkr_engine* e) { return 2 * dev::kProbeHeads * (int)(e->D + 1) * 8; }

// decode and combine are launched with programmatic dependent launch: their
// CTAs become resident while the previous kernel drains and block in
// griddepcontrol.wait until its results are visible.
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <int D>
void launch_decode(sinkr_engine* e, const dev::DevTables& t) {
    launch_pdl(dev::decode_kernel<D>, dim3(e->grid), dim3(dev::kThreads), smem_bytes<D>(),
               e->stream, e->tmk, e->tmv, t);
}

void launch_combine(sinkr_engine* e, const dev::DevTables& t, const float* src, size_t ustride,
                    size_t sstride, uint32_t fixed_n, float* dst, int mode, size_t max_n) {
    launch_pdl(dev::combine_kernel, dim3((unsigned)e->U, (unsigned)e->r, (unsigned)(e->D / 32)),
               dim3(32 * dev::kCombineGroups), max_n * 4, e->stream, t, src, (uint32_t)ustride,
               (uint32_t)sstride, fixed_n, dst, mode);
}

// Enqueues probe -> decode -> combine on the engine stream (graph-captured).
// SINKR_DEBUG_KERNELS (bitmask probe=1, decode=2, combine=4; default 7) lets a
// profiling run drop kernels from the step to attribute fixed costs.  Results
// are meaningless unless all three run; never set it outside profiling.
static int debug_kernel_mask() {
    static int m = [] {
        const char* v = std::getenv("SINKR_DEBUG_KERNELS");
        return v ? std::atoi(v) : 7;
    }();
    return m;
}

// the step-kernel instantiation of this engine (lean: single-sequence shapes;
// wide: GQA width 9-16)
using StepFn = void (*)(const dev::StepTables, const dev::ProbeParams);
template <int D>
StepFn step_fn_d(const sinkr_engine* e) {
    if (e->wide) return e->lean ? dev::step_kernel<D, true, true> : dev::step_kernel<D, false, true>;
    return e->lean ? dev::step_kernel<D, true, false> : dev::step_kernel<D, false, false>;
}
const void* step_fn(const sinkr_engine* e) {
    switch (e->D) {
        case 32: return (const void*)step_fn_d<32>(e);
        case 64: return (const void*)step_fn_d<64>(e);
        default: return (const void*)step_fn_d<128>(e);
    }
}

static int step_launch_mode() {
    static int m = [] {
        const char* v = std::getenv("SINKR_STEP_LAUNCH");
        return v ? std::atoi(v) : 0;
    }();
    return m;
}
// SINKR_STEP_GRAPH=0: device-buffer steps launch the kernel directly instead
// of replaying a captured graph (A/B knob)
static bool step_graph() {
    static bool g = [] {
        const char* v = std::getenv("SINKR_STEP_GRAPH");
        return !(v && v[0] == '0');
    }();
    return g;
}

template <int D>
void launch_step(sinkr_engine* e, const dev::StepTables& st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(e->grid);
    cfg.blockDim = dim3(dev::kThreads);
    cfg.dynamicSmemBytes = dev::StepCfg<D>::kSmemBytes;
    cfg.stream = e->stream;
    // cooperative: the merge phase waits on other CTAs, so all must be resident
    // (SINKR_STEP_LAUNCH=1 plain, =2 programmatic serialization, =3 both
    // cooperative and programmatic: A/B knobs)
    cudaLaunchAttribute attr[2];
    const int lm = step_launch_mode();
    int na = 0;
    if (lm == 0 || lm == 1 || lm == 3) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na++].val.cooperative = lm == 1 ? 0 : 1;
    }
    if (lm >= 2) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CK(cudaLaunchKernelEx(&cfg, step_fn_d<D>(e), st, e->pp));
}

void enqueue_step(sinkr_engine* e, const float* d_q, float* d_out, int mode,
                  uint8_t* res = nullptr, uint32_t* done = nullptr) {
    if (e->fused) {
        dev::StepTables st = e->step_tables(d_q, d_out, mode, res);
        st.done = done;
        if (e->timing) CK(cudaEventRecord(e->ev[0], e->stream));
        switch (e->D) {
            case 32: launch_step<32>(e, st); break;
            case 64: launch_step<64>(e, st); break;
            default: launch_step<128>(e, st); break;
        }
        if (e->timing) CK(cudaEventRecord(e->ev[3], e->stream));
        CK(cudaGetLastError());
        return;
    }
    const dev::DevTables t = e->tables(d_q);
    const int km = debug_kernel_mask();
    if (e->timing) CK(cudaEventRecord(e->ev[0], e->stream));
    if (km & 1) switch (e->D) {
        case 32: dev::probe_kernel<32><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
        case 64: dev::probe_kernel<64><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
        default: dev::probe_kernel<128><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
    }
    if (e->timing) CK(cudaEventRecord(e->ev[1], e->stream));
    if (km & 2) switch (e->D) {
        case 32: launch_decode<32>(e, t); break;
        case 64: launch_decode<64>(e, t); break;
        default: launch_decode<128>(e, t); break;
    }
    if (e->timing) CK(cudaEventRecord(e->ev[2], e->stream));
    if (km & 4) launch_combine(e, t, e->d_partials, e->S * e->PS, e->PS, 0u, d_out, mode, e->S);
    if (e->timing) CK(cudaEventRecord(e->ev[3], e->stream));
    CK(cudaGetLastError());
}

// Timing mode launches the three kernels eagerly with events between them
// (per-phase seconds, like the reference's phase timers).  Otherwise the step
// is one CUDA-graph replay, bracketed by events outside the graph.
void run_graph(sinkr_engine* e, const float* d_q, float* d_out, int mode) {
    e->last_launches = e->fused ? 1 : 3;
    e->last_mode = mode;
    if (e->timing || (e->fused && !step_graph())) {
        enqueue_step(e, d_q, d_out, mode);
        return;
    }
    const auto key = std::make_tuple((const void*)d_q, (void*)d_out, mode);
    auto it = e->graphs.find(key);
    if (it == e->graphs.end()) {
        sinkr_engine::GraphEntry ge;
        CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_step(e, d_q, d_out, mode);
        } catch (...) {
            cudaStreamEndCapture(e->stream, &ge.graph);
            if (ge.graph) cudaGraphDestroy(ge.graph);
            throw;
        }
        CK(cudaStreamEndCapture(e->stream, &ge.graph));
        CK(cudaGraphInstantiate(&ge.exec, ge.graph, 0));
        // the probe node: its by-value ProbeParams are patched every step
        size_t n = 0;
        CK(cudaGraphGetNodes(ge.graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        CK(cudaGraphGetNodes(ge.graph, nodes.data(), &n));
        const void* probe_fn =
            e->fused ? step_fn(e)
                     : (e->D == 32 ? (const void*)dev::probe_kernel<32>
                        : e->D == 64 ? (const void*)dev::probe_kernel<64>
                                     : (const void*)dev::probe_kernel<128>);
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func == probe_fn) {
                ge.probe = nd;
                ge.probe_kp = kp;
            }
        }
        if (!ge.probe && (debug_kernel_mask() & 1))
            fail(SINKR_CUDA_ERROR, "probe node not found in the captured graph");
        ge.probe_t = e->tables(d_q);
        ge.step_t = e->step_tables(d_q, d_out, mode);
        ge.fused = e->fused;
        ge.pp = e->pp;
        it = e->graphs.emplace(key, ge).first;
    }
    auto& ge = it->second;
    if (ge.probe && std::memcmp(&ge.pp, &e->pp, sizeof(e->pp)) != 0) {
        ge.pp = e->pp;
        void* args3[2] = {&ge.probe_t, &ge.pp};
        void* args1[2] = {&ge.step_t, &ge.pp};
        cudaKernelNodeParams kp = ge.probe_kp;
        kp.kernelParams = ge.fused ? args1 : args3;
        kp.extra = nullptr;
        CK(cudaGraphExecKernelNodeSetParams(ge.exec, ge.probe, &kp));
    }
    // no event records around replays unless asked: each is an extra stream
    // operation between back-to-back steps
    if (e->step_events) CK(cudaEventRecord(e->ev[0], e->stream));
    CK(cudaGraphLaunch(ge.exec, e->stream));
    if (e->step_events) CK(cudaEventRecord(e->ev[3], e->stream));
}

// The host-buffer step (sinkr_routed_decode_batch) as ONE graph: the H2D copy
// of the staged input block (params + queries) and the fused step kernel,
// which writes outputs and the routing record straight into the mapped pinned
// result block (zero-copy, no D2H copy node).  One submission per step and no
// host round trip between the copy and the kernel.
static int io_mode() {
    static int m = [] {
        const char* v = std::getenv("SINKR_IO");
        return v ? std::atoi(v) : 1;
    }();
    return m;
}

void launch_append(sinkr_engine* e, size_t layer, const float* dk, const float* dv) {
    dev::append_token_kernel<<<(unsigned)e->U, (unsigned)std::min<size_t>(e->D, 128), 0, e->stream>>>(
        dk, dv, e->d_k, e->d_v, e->d_len, (uint32_t)(layer * e->U), (uint32_t)e->D, (uint32_t)e->cap);
    CK(cudaGetLastError());
}

// The staged input block [0, bytes) to d_in, in stream order, by the upload
// kernel (a graph node ~8 us shorter than a memcpy node).
void launch_upload(sinkr_engine* e, size_t bytes) {
    const uint32_t n16 = (uint32_t)((bytes + 15) / 16);
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>((n16 + 255) / 256, (uint32_t)e->num_sms));
    dev::upload_kernel<<<grid, 256, 0, e->stream>>>(reinterpret_cast<const uint4*>(e->h_in_dev),
                                                     reinterpret_cast<uint4*>(e->d_in), n16);
    CK(cudaGetLastError());
}

// append_layer >= 0: the graph also carries the new token's K/V rows (staged
// after the queries) and appends them to every slot of that layer before
// the step (sinkr_decode_append_step)
void run_io_graph(sinkr_engine* e, int mode = 0, long append_layer = -1) {
    e->last_launches = append_layer >= 0 ? 2 : 1;
    e->last_mode = mode;
    const int code = (mode == 3 ? 6 : 2) + (append_layer >= 0 ? 1000 + 16 * (int)append_layer : 0);
    const auto key = std::make_tuple((const void*)e->h_in, (void*)e->h_res, code);
    auto it = e->graphs.find(key);
    const float* d_q = reinterpret_cast<const float*>(e->d_in + e->off_q);
    const bool zc = io_mode() == 1;
    uint8_t* res = zc ? e->h_res_dev : e->d_res;
    float* out = reinterpret_cast<float*>(res);
    if (!step_graph()) {  // A/B: the same launches without a graph
        if (zc) *reinterpret_cast<volatile uint32_t*>(e->h_done) = 0u;
        launch_upload(e, append_layer >= 0 ? e->in_bytes_append : e->in_bytes);
        if (append_layer >= 0) {
            const float* kn = reinterpret_cast<const float*>(e->d_in + e->off_kvn);
            launch_append(e, (size_t)append_layer, kn, kn + e->U * e->D);
        }
        const bool timing = e->timing;
        e->timing = false;
        enqueue_step(e, d_q, out, mode, res, zc ? e->h_done_dev : nullptr);
        e->timing = timing;
        if (!zc) CK(cudaMemcpyAsync(e->h_res, e->d_res, e->res_bytes, cudaMemcpyDeviceToHost, e->stream));
        return;
    }
    if (it == e->graphs.end()) {
        sinkr_engine::GraphEntry ge;
        CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        try {
            launch_upload(e, append_layer >= 0 ? e->in_bytes_append : e->in_bytes);
            if (append_layer >= 0) {
                const float* kn = reinterpret_cast<const float*>(e->d_in + e->off_kvn);
                launch_append(e, (size_t)append_layer, kn, kn + e->U * e->D);
            }
            const bool timing = e->timing;
            e->timing = false;
            enqueue_step(e, d_q, out, mode, res, zc ? e->h_done_dev : nullptr);
            e->timing = timing;
            if (!zc)
                CK(cudaMemcpyAsync(e->h_res, e->d_res, e->res_bytes, cudaMemcpyDeviceToHost, e->stream));
        } catch (...) {
            cudaStreamEndCapture(e->stream, &ge.graph);
            if (ge.graph) cudaGraphDestroy(ge.graph);
            throw;
        }
        CK(cudaStreamEndCapture(e->stream, &ge.graph));
        CK(cudaGraphInstantiate(&ge.exec, ge.graph, 0));
        size_t n = 0;
        CK(cudaGraphGetNodes(ge.graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        CK(cudaGraphGetNodes(ge.graph, nodes.data(), &n));
        const void* sfn = step_fn(e);
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func != sfn) continue;
            ge.probe_kp = kp;
            ge.probe = nd;
        }
        if (!ge.probe) fail(SINKR_CUDA_ERROR, "step node not found in the captured graph");
        ge.step_t = e->step_tables(d_q, out, mode, res);
        ge.step_t.done = zc ? e->h_done_dev : nullptr;
        ge.fused = true;
        ge.pp = e->pp;
        it = e->graphs.emplace(key, ge).first;
    }
    auto& ge = it->second;
    if (std::memcmp(&ge.pp, &e->pp, sizeof(e->pp)) != 0) {
        ge.pp = e->pp;
        void* args[2] = {&ge.step_t, &ge.pp};
        cudaKernelNodeParams kp = ge.probe_kp;
        kp.kernelParams = args;
        kp.extra = nullptr;
        CK(cudaGraphExecKernelNodeSetParams(ge.exec, ge.probe, &kp));
    }
    if (zc) *reinterpret_cast<volatile uint32_t*>(e->h_done) = 0u;
    CK(cudaGraphLaunch(ge.exec, e->stream));
}

// Waits for a step launched by run_io_graph.  With zero-copy results the
// step kernel's last CTA sets the completion word after a system-scope
// fence, so the host spins on that word (it sees the results as soon as the
// last CTA has written them, without the kernel-retire -> stream-sync round
// trip); the stream is polled now and then so a failed launch cannot hang.
void finish_io(sinkr_engine* e) {
    if (io_mode() != 1) {
        CK(cudaStreamSynchronize(e->stream));
        return;
    }
    const volatile uint32_t* w = e->h_done;
    for (uint32_t i = 1;; ++i) {
        if (*w) break;
        if ((i & 0x3FFFu) == 0) {
            const cudaError_t q = cudaStreamQuery(e->stream);
            if (q == cudaSuccess) {
                if (*w) break;
                fail(SINKR_CUDA_ERROR, "step finished without setting its completion word");
            }
            if (q != cudaErrorNotReady) CK(q);
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
}

size_t token_count(const sinkr_engine* e, size_t seq) {
    const size_t H = e->cfg.num_kv_heads;
    const size_t n = e->len[e->slot_index(0, seq, 0)];
    for (size_t l = 0; l < e->layers; ++l)
        for (size_t g = 0; g < H; ++g)
            if (e->len[e->slot_index(l, seq, g)] != n)
                fail(SINKR_LOGIC_ERROR, "kv cache lengths are ragged across slots");
    return n;
}

// Brings the device length table up to date after host-path appends (the
// token-append kernel reads and advances it).  Host paths synchronise the
// stream when they finish, so the pinned staging is free here.
void sync_dlen(sinkr_engine* e) {
    if (!e->dlen_dirty) return;
    for (size_t i = 0; i < e->len.size(); ++i) e->h_len_stage[i] = (uint32_t)e->len[i];
    CK(cudaMemcpyAsync(e->d_len, e->h_len_stage, e->len.size() * 4, cudaMemcpyHostToDevice, e->stream));
    e->dlen_dirty = false;
}

// One new row for every (seq, kv_head) slot of `layer`: capacity checked
// first (kv_cache.cpp:67-69); true when some slot is still empty (its first
// row needs the host path: anchor capture + degenerate check).
bool check_token_append(sinkr_engine* e, size_t layer) {
    if (layer >= e->layers) fail(SINKR_OUT_OF_RANGE, "layer index out of range");
    bool empty = false;
    for (size_t u = 0; u < e->U; ++u) {
        const size_t n = e->len[layer * e->U + u];
        if (n + 1 > e->cap)
            fail(SINKR_RUNTIME_ERROR, "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        empty |= n == 0;
    }
    return empty;
}

// Validates a step (router.cpp:85-90) and stages hdr / tau / len into the
// pinned input block; uploads them only when they changed.
// the pinned input block is free once the last copy out of it ran (the
// one-graph host-buffer path needs no event: the call returns after its step)
void wait_input_block(sinkr_engine* e) {
    if (!e->ev_in_pending) return;
    CK(cudaEventSynchronize(e->ev_in));
    e->ev_in_pending = false;
}

void stage_params(sinkr_engine* e, size_t layer, const sinkr_routing_config* cfg,
                  const sinkr_engine_options* opt, bool defer_upload) {
    if (!cfg) fail(SINKR_INVALID_ARGUMENT, "routing config is null");
    if (layer >= e->layers) fail(SINKR_OUT_OF_RANGE, "layer index out of range");
    sinkr_engine_options o{};
    o.block_size = dev::kStageTok;
    if (opt) o = *opt;
    // wait until the previous upload consumed the pinned staging block
    wait_input_block(e);
    auto* hdr = reinterpret_cast<dev::StepHdr*>(e->h_in);
    auto* tau = reinterpret_cast<double*>(e->h_in + e->off_tau);
    auto* len = reinterpret_cast<uint32_t*>(e->h_in + e->off_len);
    hdr->layer = (uint32_t)layer;
    hdr->flags = (o.observe_only ? dev::kObserveOnly : 0u) |
                 (cfg->sink_on_tie ? dev::kSinkOnTie : 0u) |
                 (layer_excluded(layer, *cfg) ? dev::kLayerExcluded : 0u);
    hdr->pad[0] = hdr->pad[1] = 0;
    for (size_t s = 0; s < e->B; ++s) {
        const size_t L = token_count(e, s);
        if (L == 0) fail(SINKR_RUNTIME_ERROR, "routed decode over an empty cache");
        for (size_t g = 0; g < e->cfg.num_kv_heads; ++g)
            if (!e->anchored[e->slot_index(layer, s, g)])
                fail(SINKR_RUNTIME_ERROR, "anchor requested from empty cache slot");
        const size_t Lg = o.global_context_len ? o.global_context_len : L;
        tau[s] = threshold_for_length(Lg, cfg->profile);
        len[s] = (uint32_t)L;
    }
    std::memset(&e->pp, 0, sizeof(e->pp));
    e->pp.layer = hdr->layer;
    e->pp.flags = hdr->flags;
    e->pp.inline_seqs = e->B <= (size_t)dev::kParamSeqs ? 1u : 0u;
    if (e->pp.inline_seqs)
        for (size_t s = 0; s < e->B; ++s) {
            e->pp.tau[s] = tau[s];
            e->pp.len[s] = len[s];
        }
    const size_t pbytes = e->off_q;
    const bool same = e->params_valid && e->last_params.size() == pbytes &&
                      std::memcmp(e->last_params.data(), e->h_in, pbytes) == 0;
    if (!defer_upload && !same) {
        CK(cudaMemcpyAsync(e->d_in, e->h_in, pbytes, cudaMemcpyHostToDevice, e->stream));
        CK(cudaEventRecord(e->ev_in, e->stream));
        e->ev_in_pending = true;
    }
    e->last_params.assign(e->h_in, e->h_in + pbytes);
    e->params_valid = true;
}

void fill_info(sinkr_engine* e, size_t layer, const sinkr_routing_config* cfg,
               sinkr_group_info* groups, double* head_scores, sinkr_load_counters* counters,
               const sinkr_engine_options* opt) {
    const size_t H = e->cfg.num_kv_heads, Hq = e->cfg.num_q_heads;
    const auto* hs = reinterpret_cast<const double*>(e->h_res + e->off_hs);
    const auto* gs = reinterpret_cast<const double*>(e->h_res + e->off_gs);
    const auto* tok = reinterpret_cast<const unsigned long long*>(e->h_res + e->off_tok);
    const auto* fl = reinterpret_cast<const uint32_t*>(e->h_res + e->off_fl);
    const auto* tau = reinterpret_cast<const double*>(e->h_in + e->off_tau);
    sinkr_load_counters c{};
    for (size_t u = 0; u < e->U; ++u) {
        const size_t s = u / H;
        if (groups) {
            sinkr_group_info& gi = groups[u];
            gi.layer = layer;
            gi.kv_head = u % H;
            gi.group_score = gs[u];
            gi.threshold = tau[s];
            gi.sink = (fl[u] & dev::kSink) ? 1 : 0;
            gi.degenerate = (fl[u] & dev::kDegenerate) ? 1 : 0;
            gi.tokens_loaded = tok[u];
            gi.kv_floats_loaded = 2ull * tok[u] * e->D;
        }
        c.kv_floats_loaded += 2ull * tok[u] * e->D;
        if (fl[u] & dev::kActive)
            ++c.groups_active;
        else
            ++c.groups_skipped;
    }
    c.anchor_floats_loaded = (uint64_t)(e->U * e->D);
    if (head_scores) std::memcpy(head_scores, hs, e->B * Hq * sizeof(double));
    if (e->fused) {
        // device-side phase stamps (%globaltimer, ns) written by the step kernel
        const auto* st = reinterpret_cast<const uint32_t*>(e->h_res + e->off_status);
        const auto* clk = reinterpret_cast<const unsigned long long*>(st + 4);
        if (st[0]) {
            if (st[0] == 5) e->peer_poisoned = true;
            static const char* what[] = {"", "partial spill-slot lock timeout",
                                         "merge watchdog: a group never completed",
                                         "routing grid-barrier watchdog",
                                         "fp32 route estimate disagreed with the exact route",
                                         "peer merge watchdog: a rank never delivered its partials"};
            fail(SINKR_RUNTIME_ERROR, std::string("step kernel error: ") + (st[0] < 6 ? what[st[0]] : "unknown"));
        }
        if (clk[1] >= clk[0] && clk[2] >= clk[1] && clk[3] >= clk[2]) {
            c.routing_seconds = (clk[1] - clk[0]) * 1e-9;
            c.attention_seconds = (clk[2] - clk[1]) * 1e-9;
            c.merge_seconds = (clk[3] - clk[2]) * 1e-9;
        }
    } else if (e->timing) {
        float ms[3] = {0, 0, 0};
        for (int i = 0; i < 3; ++i) CK(cudaEventElapsedTime(&ms[i], e->ev[i], e->ev[i + 1]));
        c.routing_seconds = ms[0] * 1e-3;
        c.attention_seconds = ms[1] * 1e-3;
        c.merge_seconds = ms[2] * 1e-3;
    }
    if (counters) *counters = c;
    (void)cfg;
    // attend_chunk rejects block_size == 0 only when a group actually runs
    // (attention.cpp:297), so the check happens after routing.
    if (opt && opt->block_size == 0 && c.groups_active > 0)
        fail(SINKR_INVALID_ARGUMENT, "block_size must be positive");
}

void check_error_flag(sinkr_engine* e) {
    dev::WorkState ws;
    CK(cudaMemcpyAsync(&ws, e->d_ws, sizeof(ws), cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    if (ws.error) fail(SINKR_RUNTIME_ERROR, "decode partial-slot overflow");
}

void upload_anchor(sinkr_engine* e, size_t idx) {
    CK(cudaMemcpyAsync(e->d_anchor + idx * e->D, e->h_anchor.data() + idx * e->D, e->D * 4,
                       cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(e->d_anchor_norm + idx, e->h_anchor_norm.data() + idx, 4,
                       cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
}

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================
extern "C" {

const char* sinkr_last_error(void) { return g_err.c_str(); }
const char* sinkr_version(void) { return "sinkr-b200 0.1 (sm_100a)"; }

sinkr_status sinkr_engine_create(const sinkr_cache_config* config, int device,
                                 sinkr_engine** out) {
    return guard([&] {
        if (!config || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const sinkr_cache_config& c = *config;
        // CacheConfig::validate (kv_cache.cpp:32-39)
        if (c.num_layers == 0) fail(SINKR_INVALID_ARGUMENT, "num_layers must be positive");
        if (c.num_kv_heads == 0) fail(SINKR_INVALID_ARGUMENT, "num_kv_heads must be positive");
        if (c.num_q_heads == 0 || c.num_q_heads % c.num_kv_heads != 0)
            fail(SINKR_INVALID_ARGUMENT, "num_q_heads must be a positive multiple of num_kv_heads");
        if (c.head_dim == 0) fail(SINKR_INVALID_ARGUMENT, "head_dim must be positive");
        if (c.capacity == 0) fail(SINKR_INVALID_ARGUMENT, "capacity must be positive");
        if (c.head_dim != 32 && c.head_dim != 64 && c.head_dim != 128)
            fail(SINKR_INVALID_ARGUMENT, "head_dim must be 32, 64 or 128 on the GPU engine");
        if (c.num_q_heads / c.num_kv_heads > (size_t)dev::kMaxRWide)
            fail(SINKR_INVALID_ARGUMENT, "GQA group width above 16 is not supported");

        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            fail(SINKR_NO_DEVICE, "no CUDA device visible (the engine has no CPU fallback)");
        }
        if (device < 0 || device >= ndev) fail(SINKR_NO_DEVICE, "device ordinal out of range");
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10)
            fail(SINKR_NO_DEVICE, std::string("sm_100 device required, found ") + prop.name);
        CK(cudaSetDevice(device));

        auto* e = new sinkr_engine();
        try {
            e->cfg = c;
            e->B = c.num_seqs ? c.num_seqs : 1;
            e->cfg.num_seqs = e->B;
            e->U = e->B * c.num_kv_heads;
            e->r = c.num_q_heads / c.num_kv_heads;
            e->D = c.head_dim;
            e->layers = c.num_layers;
            e->cap = c.capacity;
            e->device = device;
            e->num_sms = prop.multiProcessorCount;
            e->grid = e->num_sms;
            // SINKR_DEBUG_GRID: fewer persistent CTAs (tests run two engines'
            // cooperative kernels side by side on one GPU)
            if (const char* dg = std::getenv("SINKR_DEBUG_GRID"); dg && std::atoi(dg) > 0)
                e->grid = std::min(e->grid, std::atoi(dg));
            const size_t rows = e->layers * e->B * c.num_kv_heads * e->cap;
            if (rows >= (size_t(1) << 31))
                fail(SINKR_INVALID_ARGUMENT, "cache exceeds 2^31 rows (TMA coordinate range)");
            CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
            const size_t kv_bytes = rows * e->D * 2;
            CK(cudaMalloc(&e->d_k, kv_bytes));
            CK(cudaMalloc(&e->d_v, kv_bytes));
            // rows past a slot's length are read (and masked) by tail stages:
            // keep them finite.
            CK(cudaMemsetAsync(e->d_k, 0, kv_bytes, e->stream));
            CK(cudaMemsetAsync(e->d_v, 0, kv_bytes, e->stream));
            const size_t slots = e->layers * e->B * c.num_kv_heads;
            CK(cudaMalloc(&e->d_anchor, slots * e->D * 4));
            CK(cudaMalloc(&e->d_anchor_norm, slots * 4));
            CK(cudaMalloc(&e->d_norm64, 8));
            CK(cudaMemsetAsync(e->d_anchor, 0, slots * e->D * 4, e->stream));
            CK(cudaMemsetAsync(e->d_anchor_norm, 0, slots * 4, e->stream));
            e->len.assign(slots, 0);
            e->h_anchor.assign(slots * e->D, 0.f);
            e->h_anchor_norm.assign(slots, 0.f);
            e->anchored.assign(slots, 0);

            const size_t Hq = c.num_q_heads;
            e->off_tau = 64;
            e->off_len = align_up(e->off_tau + 8 * e->B, 64);
            e->off_q = align_up(e->off_len + 4 * e->B, 128);
            e->in_bytes = e->off_q + e->B * Hq * e->D * 4;
            e->off_kvn = align_up(e->in_bytes, 128);
            e->in_bytes_append = e->off_kvn + 2 * e->U * e->D * 4;
            CK(cudaMalloc(&e->d_in, e->in_bytes_append));
            CK(cudaHostAlloc(&e->h_in, e->in_bytes_append, cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_in_dev), e->h_in, 0));
            std::memset(e->h_in, 0, e->in_bytes_append);
            CK(cudaMalloc(&e->d_len, slots * 4));
            CK(cudaMemsetAsync(e->d_len, 0, slots * 4, e->stream));
            CK(cudaMallocHost(&e->h_len_stage, slots * 4));

            e->off_hs = align_up(e->B * Hq * e->D * 4, 128);
            e->off_gs = align_up(e->off_hs + e->B * Hq * 8, 128);
            e->off_tok = align_up(e->off_gs + e->U * 8, 128);
            e->off_fl = align_up(e->off_tok + e->U * 8, 128);
            e->off_status = align_up(e->off_fl + e->U * 4, 128);  // status[4] + clocks
            e->res_bytes = align_up(e->off_status + 64 + 256, 128);
            CK(cudaMalloc(&e->d_res, e->res_bytes));
            CK(cudaHostAlloc(&e->h_res, e->res_bytes, cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_res_dev), e->h_res, 0));
            std::memset(e->h_res, 0, e->res_bytes);
            CK(cudaMemsetAsync(e->d_res, 0, e->res_bytes, e->stream));
            CK(cudaHostAlloc(reinterpret_cast<void**>(&e->h_done), 64, cudaHostAllocMapped));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_done_dev), e->h_done, 0));
            *e->h_done = 0u;

            CK(cudaMalloc(&e->d_head_degen, e->B * Hq * 4));
            e->probe_grid = (int)((e->B * Hq + dev::kProbeHeads - 1) / dev::kProbeHeads);
            // the step kernel's lean routing form (step.cuh): every single-sequence shape
            e->lean = e->B * Hq <= (size_t)dev::kRouteTile && e->U <= 32;
            e->wide = e->r > (size_t)dev::kMaxR;
            CK(cudaMalloc(&e->d_ss, sizeof(dev::StepState)));
            CK(cudaMemsetAsync(e->d_ss, 0, sizeof(dev::StepState), e->stream));
            // per-unit step counters: two sets, used by alternate launches
            // (StepCounters, step.cuh); the per-CTA launch counts pick the set
            CK(cudaMalloc(&e->d_cursor, 2 * e->U * 4));
            CK(cudaMemsetAsync(e->d_cursor, 0, 2 * e->U * 4, e->stream));
            CK(cudaMalloc(&e->d_tokens_done, 2 * e->U * 4));
            CK(cudaMalloc(&e->d_route_flags, e->U * 4));
            CK(cudaMalloc(&e->d_ovf, 2 * e->U * 4));
            CK(cudaMemsetAsync(e->d_ovf, 0, 2 * e->U * 4, e->stream));
            CK(cudaMemsetAsync(e->d_tokens_done, 0, 2 * e->U * 4, e->stream));
            CK(cudaMalloc(&e->d_route_sum, e->grid * 4));
            CK(cudaMalloc(&e->d_spec_mask, e->layers * 4));
            CK(cudaMemsetAsync(e->d_spec_mask, 0, e->layers * 4, e->stream));
            CK(cudaMalloc(&e->d_cta_epoch, 2 * e->grid * 4));  // launches, mode-3 steps
            CK(cudaMemsetAsync(e->d_cta_epoch, 0, 2 * e->grid * 4, e->stream));
            if (const char* tr = std::getenv("SINKR_TRACE"); tr && tr[0] == '1') {
                CK(cudaMalloc(&e->d_trace, e->grid * 8 * 8));
                CK(cudaMemsetAsync(e->d_trace, 0, e->grid * 8 * 8, e->stream));
            }
            {
                const char* f = std::getenv("SINKR_FUSED");
                const bool fits = e->U <= (size_t)dev::kMaxUnits && e->B * Hq <= (size_t)dev::kMaxStepHeads;
                // (the three-kernel A/B pipeline holds one 8-head tile per group)
                e->fused = fits && (e->wide || !(f && f[0] == '0'));
                if (e->wide && !fits)
                    fail(SINKR_INVALID_ARGUMENT, "GQA group width above 8 needs B*H_kv <= 1280 and B*H_q <= 4096");
            }
            CK(cudaMalloc(&e->d_ws, sizeof(dev::WorkState)));
            CK(cudaMemsetAsync(e->d_ws, 0, sizeof(dev::WorkState), e->stream));
            CK(cudaMalloc(&e->d_active, e->U * 16));
            CK(cudaMalloc(&e->d_prefix, (e->U + 1) * 4));  // unit_next cursors
            CK(cudaMalloc(&e->d_slot_count, 2 * e->U * 4));
            CK(cudaMemsetAsync(e->d_slot_count, 0, 2 * e->U * 4, e->stream));
            // partial slots per unit: one per (CTA, unit) visit up to S-1; any
            // further partial of a unit is LSE-combined into slot S-1 under a
            // per-unit lock (step.cuh flush), so S only sizes the fast path.
            // SINKR_DEBUG_SLOTS forces a small S to exercise the spill path.
            e->S = std::min<size_t>(e->grid, (e->cap + dev::kStageTok - 1) / dev::kStageTok) + 32;
            if (const char* ds = std::getenv("SINKR_DEBUG_SLOTS"); ds && std::atoi(ds) >= 2)
                e->S = (size_t)std::atoi(ds);
            // even: a unit's slot block then starts 16-byte aligned (PS is
            // even), which the merge's bulk copies need
            e->S = (e->S + 1) & ~size_t(1);
            e->PS = e->r * (e->D + 2);
            // + 64 slots: warp_merge loads groups of 64 slots unpredicated
            CK(cudaMalloc(&e->d_partials, (e->U * e->S + 64) * e->PS * 4));
            // combine reads candidate slots speculatively: keep them finite
            CK(cudaMemsetAsync(e->d_partials, 0, (e->U * e->S + 64) * e->PS * 4, e->stream));

            make_tmap(&e->tmk, e->d_k, rows, e->D);
            make_tmap(&e->tmv, e->d_v, rows, e->D);
            CK(cudaMalloc(&e->d_tmap, 2 * sizeof(CUtensorMap)));
            CUtensorMap both[2] = {e->tmk, e->tmv};
            CK(cudaMemcpy(e->d_tmap, both, sizeof(both), cudaMemcpyHostToDevice));
            CK(cudaFuncSetAttribute(dev::decode_kernel<32>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<32>()));
            CK(cudaFuncSetAttribute(dev::decode_kernel<64>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<64>()));
            CK(cudaFuncSetAttribute(dev::decode_kernel<128>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_bytes<128>()));
            for (int nt = 1; nt <= 2; ++nt) {
                CK(cudaFuncSetAttribute(nt == 1 ? (const void*)dev::bos_stream_kernel<32, 1>
                                                : (const void*)dev::bos_stream_kernel<32, 2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, dev::BosCfg<32>::kSmemBytes));
                CK(cudaFuncSetAttribute(nt == 1 ? (const void*)dev::bos_stream_kernel<64, 1>
                                                : (const void*)dev::bos_stream_kernel<64, 2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, dev::BosCfg<64>::kSmemBytes));
                CK(cudaFuncSetAttribute(nt == 1 ? (const void*)dev::bos_stream_kernel<128, 1>
                                                : (const void*)dev::bos_stream_kernel<128, 2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, dev::BosCfg<128>::kSmemBytes));
            }
            CK(cudaFuncSetAttribute(step_fn(e), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    e->D == 32 ? dev::StepCfg<32>::kSmemBytes
                                    : e->D == 64 ? dev::StepCfg<64>::kSmemBytes
                                                 : dev::StepCfg<128>::kSmemBytes));
            CK(cudaFuncSetAttribute(dev::probe_kernel<32>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, probe_smem(e)));
            CK(cudaFuncSetAttribute(dev::probe_kernel<64>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, probe_smem(e)));
            CK(cudaFuncSetAttribute(dev::probe_kernel<128>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, probe_smem(e)));
            for (const void* fn : {(const void*)dev::score_batch_kernel<32>, (const void*)dev::score_batch_kernel<64>,
                                   (const void*)dev::score_batch_kernel<128>})
                CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        2 * dev::kScoreHeads * (int)(e->D + 1) * 8));
            // one shared-memory carveout for all step kernels: switching the
            // L1/smem split between back-to-back kernels stalls the SMs
            for (const void* fn : {(const void*)dev::probe_kernel<32>, (const void*)dev::probe_kernel<64>,
                                   (const void*)dev::probe_kernel<128>, (const void*)dev::combine_kernel,
                                   (const void*)dev::decode_kernel<32>, (const void*)dev::decode_kernel<64>,
                                   (const void*)dev::decode_kernel<128>})
                CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared));
            for (auto& ev : e->ev) CK(cudaEventCreate(&ev));
            CK(cudaEventCreateWithFlags(&e->ev_in, cudaEventDisableTiming));
            CK(cudaEventCreate(&e->ev_bos[0]));
            CK(cudaEventCreate(&e->ev_bos[1]));
            CK(cudaEventRecord(e->ev_in, e->stream));
            e->ev_in_pending = true;
            CK(cudaStreamSynchronize(e->stream));
        } catch (...) {
            sinkr_engine_destroy(e);
            throw;
        }
        *out = e;
    });
}

sinkr_status sinkr_engine_destroy(sinkr_engine* e) {
    if (!e) return SINKR_OK;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (auto& kv : e->graphs) {
        cudaGraphExecDestroy(kv.second.exec);
        cudaGraphDestroy(kv.second.graph);
    }
    e->drop_bos_graphs();
    for (auto& ev : e->ev)
        if (ev) cudaEventDestroy(ev);
    if (e->ev_in) cudaEventDestroy(e->ev_in);
    cudaFree(e->d_k);
    cudaFree(e->d_v);
    cudaFree(e->d_anchor);
    cudaFree(e->d_anchor_norm);
    cudaFree(e->d_norm64);
    cudaFree(e->d_in);
    cudaFree(e->d_res);
    cudaFree(e->d_ws);
    cudaFree(e->d_ss);
    cudaFree(e->d_tmap);
    cudaFree(e->d_cursor);
    cudaFree(e->d_tokens_done);
    cudaFree(e->d_route_flags);
    cudaFree(e->d_bos);
    cudaFree(e->d_span);
    for (void* pb : e->ipc_opened) cudaIpcCloseMemHandle(pb);
    cudaFree(e->d_xchg);
    cudaFree(e->d_peer_xchg);
    cudaFree(e->d_ovf);
    cudaFree(e->d_cta_epoch);
    cudaFree(e->d_spec_mask);
    cudaFree(e->d_route_sum);
    cudaFree(e->d_head_degen);
    cudaFree(e->d_active);
    cudaFree(e->d_prefix);
    cudaFree(e->d_slot_count);
    cudaFree(e->d_partials);
    if (e->h_in) cudaFreeHost(e->h_in);
    if (e->h_res) cudaFreeHost(e->h_res);
    if (e->h_done) cudaFreeHost(e->h_done);
    if (e->d_score_scratch) cudaFree(e->d_score_scratch);
    if (e->h_len_stage) cudaFreeHost(e->h_len_stage);
    cudaFree(e->d_len);
    if (e->h_bos) cudaFreeHost(e->h_bos);
    for (auto ev : e->ev_bos)
        if (ev) cudaEventDestroy(ev);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
    return SINKR_OK;
}

void* sinkr_engine_stream(sinkr_engine* e) { return e ? (void*)e->stream : nullptr; }
int sinkr_decode_grid(sinkr_engine* e) { return e ? e->grid : 0; }

sinkr_status sinkr_kv_append(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             const float* k, const float* v, size_t rows) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        if (rows == 0) return;
        if (!k || !v) fail(SINKR_INVALID_ARGUMENT, "k/v row size does not match head_dim");
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D;
        if (e->len[idx] + rows > e->cap)
            fail(SINKR_RUNTIME_ERROR,
                 "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        std::vector<uint16_t> kb(rows * D), vb(rows * D);
        for (size_t i = 0; i < rows * D; ++i) {
            kb[i] = f32_to_bf16(k[i]);
            vb[i] = f32_to_bf16(v[i]);
        }
        if (e->len[idx] == 0) {
            // kv_cache.cpp:71-77 on the stored (bf16-rounded) first key
            double s = 0.0;
            for (size_t j = 0; j < D; ++j) {
                const double x = bf16_to_f32(kb[j]);
                s += x * x;
            }
            const double n = std::sqrt(s);
            if (n < 1e-12)
                fail(SINKR_RUNTIME_ERROR, "degenerate anchor: first-token key norm below 1e-12");
            for (size_t j = 0; j < D; ++j) e->h_anchor[idx * D + j] = bf16_to_f32(kb[j]);
            e->h_anchor_norm[idx] = (float)n;
            upload_anchor(e, idx);
            e->anchored[idx] = 1;
        }
        const size_t off = (e->row_base(layer, seq, kv_head) + e->len[idx]) * D;
        CK(cudaMemcpyAsync(e->d_k + off, kb.data(), rows * D * 2, cudaMemcpyHostToDevice,
                           e->stream));
        CK(cudaMemcpyAsync(e->d_v + off, vb.data(), rows * D * 2, cudaMemcpyHostToDevice,
                           e->stream));
        CK(cudaStreamSynchronize(e->stream));
        e->len[idx] += rows;
        e->dlen_dirty = true;
    });
}

static void capture_anchor_device(sinkr_engine* e, size_t idx) {
    const size_t D = e->D;
    const __nv_bfloat16* row0 = e->d_k + idx * e->cap * D;  // row 0 of the slot
    dev::anchor_capture_kernel<<<1, 32, 0, e->stream>>>(row0, (uint32_t)D, e->d_anchor + idx * D,
                                                        e->d_anchor_norm + idx, e->d_norm64);
    CK(cudaGetLastError());
    double n = 0;
    CK(cudaMemcpyAsync(&n, e->d_norm64, 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(e->h_anchor.data() + idx * D, e->d_anchor + idx * D, D * 4,
                       cudaMemcpyDeviceToHost, e->stream));
    CK(cudaMemcpyAsync(e->h_anchor_norm.data() + idx, e->d_anchor_norm + idx, 4,
                       cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    if (n < 1e-12) fail(SINKR_RUNTIME_ERROR, "degenerate anchor: first-token key norm below 1e-12");
    e->anchored[idx] = 1;
}

sinkr_status sinkr_kv_append_device_bf16(sinkr_engine* e, size_t seq, size_t layer,
                                         size_t kv_head, const void* k, const void* v,
                                         size_t rows) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        if (rows == 0) return;
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D;
        if (e->len[idx] + rows > e->cap)
            fail(SINKR_RUNTIME_ERROR,
                 "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        const size_t off = (e->row_base(layer, seq, kv_head) + e->len[idx]) * D;
        CK(cudaMemcpyAsync(e->d_k + off, k, rows * D * 2, cudaMemcpyDeviceToDevice, e->stream));
        CK(cudaMemcpyAsync(e->d_v + off, v, rows * D * 2, cudaMemcpyDeviceToDevice, e->stream));
        if (e->len[idx] == 0) capture_anchor_device(e, idx);
        CK(cudaStreamSynchronize(e->stream));
        e->len[idx] += rows;
        e->dlen_dirty = true;
    });
}

sinkr_status sinkr_kv_append_device_f32(sinkr_engine* e, size_t seq, size_t layer,
                                        size_t kv_head, const float* d_k, const float* d_v,
                                        size_t rows) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        if (rows == 0) return;
        if (!d_k || !d_v) fail(SINKR_INVALID_ARGUMENT, "k/v row size does not match head_dim");
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D;
        if (e->len[idx] + rows > e->cap)
            fail(SINKR_RUNTIME_ERROR,
                 "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        if ((reinterpret_cast<uintptr_t>(d_k) | reinterpret_cast<uintptr_t>(d_v)) & 15)
            fail(SINKR_INVALID_ARGUMENT, "device rows must be 16-byte aligned");
        const size_t off = (e->row_base(layer, seq, kv_head) + e->len[idx]) * D;
        const size_t n = rows * D;
        const int grid = (int)std::min<size_t>((n / 4 + 255) / 256 + 1, (size_t)e->num_sms * 8);
        dev::f32_to_bf16_kernel<<<grid, 256, 0, e->stream>>>(d_k, e->d_k + off, n);
        dev::f32_to_bf16_kernel<<<grid, 256, 0, e->stream>>>(d_v, e->d_v + off, n);
        CK(cudaGetLastError());
        if (e->len[idx] == 0) capture_anchor_device(e, idx);
        CK(cudaStreamSynchronize(e->stream));
        e->len[idx] += rows;
        e->dlen_dirty = true;
    });
}

sinkr_status sinkr_engine_config(sinkr_engine* e, sinkr_cache_config* out) {
    return guard([&] {
        if (!e || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        *out = e->cfg;
        out->num_seqs = e->B;
    });
}

sinkr_status sinkr_kv_append_synthetic(sinkr_engine* e, size_t seq, size_t layer,
                                       size_t kv_head, uint64_t key_k, uint64_t key_v,
                                       float k_scale, float v_scale, size_t global_row0,
                                       size_t rows) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        if (rows == 0) return;
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D;
        if (e->len[idx] + rows > e->cap)
            fail(SINKR_RUNTIME_ERROR,
                 "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        const size_t row0 = e->len[idx];
        const size_t off = (e->row_base(layer, seq, kv_head) + row0) * D;
        const uint64_t n = (uint64_t)rows * D;
        const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148ull * 64);
        dev::synth_rows_kernel<<<blocks, 256, 0, e->stream>>>(e->d_k + off, e->d_v + off, key_k,
                                                             key_v, k_scale, v_scale, global_row0,
                                                             rows, (uint32_t)D);
        CK(cudaGetLastError());
        if (row0 == 0) capture_anchor_device(e, idx);
        CK(cudaStreamSynchronize(e->stream));
        e->len[idx] += rows;
        e->dlen_dirty = true;
    });
}

sinkr_status sinkr_kv_length(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             size_t* out) {
    return guard([&] {
        if (!e || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        check_slot(e, seq, layer, kv_head);
        *out = e->len[e->slot_index(layer, seq, kv_head)];
    });
}

sinkr_status sinkr_kv_token_count(sinkr_engine* e, size_t seq, size_t* out) {
    return guard([&] {
        if (!e || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (seq >= e->B) fail(SINKR_OUT_OF_RANGE, "sequence index out of range");
        *out = token_count(e, seq);
    });
}

sinkr_status sinkr_kv_anchor(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             float* k0, float* k0_norm) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        const size_t idx = e->slot_index(layer, seq, kv_head);
        if (!e->anchored[idx]) fail(SINKR_RUNTIME_ERROR, "anchor requested from empty cache slot");
        if (k0) std::memcpy(k0, e->h_anchor.data() + idx * e->D, e->D * 4);
        if (k0_norm) *k0_norm = e->h_anchor_norm[idx];
    });
}

sinkr_status sinkr_kv_set_anchor(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                                 const float* k0, float k0_norm) {
    return guard([&] {
        if (!e || !k0) fail(SINKR_INVALID_ARGUMENT, "null argument");
        check_slot(e, seq, layer, kv_head);
        if (!(k0_norm >= 1e-12f))
            fail(SINKR_RUNTIME_ERROR, "degenerate anchor: first-token key norm below 1e-12");
        const size_t idx = e->slot_index(layer, seq, kv_head);
        std::memcpy(e->h_anchor.data() + idx * e->D, k0, e->D * 4);
        e->h_anchor_norm[idx] = k0_norm;
        upload_anchor(e, idx);
        e->anchored[idx] = 1;
    });
}

sinkr_status sinkr_kv_read(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                           size_t from, size_t to, float* k, float* v) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        check_slot(e, seq, layer, kv_head);
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D;
        if (from > to || to > e->len[idx])
            fail(SINKR_OUT_OF_RANGE, "historical range [" + std::to_string(from) + ", " +
                                         std::to_string(to) + ") exceeds length " +
                                         std::to_string(e->len[idx]));
        const size_t n = (to - from) * D;
        if (n == 0) return;
        float* tmp = nullptr;
        CK(cudaMallocAsync(&tmp, n * 4, e->stream));
        const size_t off = (e->row_base(layer, seq, kv_head) + from) * D;
        const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 32);
        for (int which = 0; which < 2; ++which) {
            float* dst = which ? v : k;
            if (!dst) continue;
            dev::upcast_kernel<<<blocks, 256, 0, e->stream>>>((which ? e->d_v : e->d_k) + off, tmp,
                                                              n);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(dst, tmp, n * 4, cudaMemcpyDeviceToHost, e->stream));
        }
        CK(cudaFreeAsync(tmp, e->stream));
        CK(cudaStreamSynchronize(e->stream));
    });
}

// ---- routing helpers ---------------------------------------------------------
sinkr_status sinkr_threshold_for_length(size_t context_len,
                                        const sinkr_threshold_profile* profile, double* out) {
    return guard([&] {
        if (!profile || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        *out = threshold_for_length(context_len, *profile);
    });
}

sinkr_status sinkr_route(size_t layer, double score, size_t context_len,
                         const sinkr_routing_config* config, int* sink, double* threshold) {
    return guard([&] {
        if (!config || !sink || !threshold) fail(SINKR_INVALID_ARGUMENT, "null argument");
        *threshold = threshold_for_length(context_len, config->profile);
        const bool over = config->sink_on_tie ? score >= *threshold : score > *threshold;
        *sink = (over && !layer_excluded(layer, *config)) ? 1 : 0;
    });
}

size_t sinkr_auto_num_splits(size_t context_len) {
    const size_t s = (context_len + 8191) / 8192;
    return std::clamp<size_t>(s, 1, 16);
}

sinkr_status sinkr_split_ranges(size_t len, size_t num_splits, size_t* from_to) {
    return guard([&] {
        if (num_splits == 0 || num_splits > len)
            fail(SINKR_INVALID_ARGUMENT, "num_splits must be in [1, len], got " +
                                             std::to_string(num_splits) + " for len " +
                                             std::to_string(len));
        if (!from_to) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const size_t base = len / num_splits, rem = len % num_splits;
        size_t start = 0;
        for (size_t c = 0; c < num_splits; ++c) {
            const size_t sz = base + (c < rem ? 1 : 0);
            from_to[2 * c] = start;
            from_to[2 * c + 1] = start + sz;
            start += sz;
        }
    });
}

// ---- hot path ------------------------------------------------------------------
static void decode_host(sinkr_engine* e, const float* queries, size_t layer,
                        const sinkr_routing_config* config, const sinkr_engine_options* options,
                        float* outputs, sinkr_group_info* groups, double* head_scores,
                        sinkr_load_counters* counters, int mode);

sinkr_status sinkr_routed_decode_batch(sinkr_engine* e, const float* queries, size_t layer,
                                       const sinkr_routing_config* config,
                                       const sinkr_engine_options* options, float* outputs,
                                       sinkr_group_info* groups, double* head_scores,
                                       sinkr_load_counters* counters) {
    return guard([&] {
        decode_host(e, queries, layer, config, options, outputs, groups, head_scores, counters, 0);
    });
}

sinkr_status sinkr_routed_decode_peer(sinkr_engine* e, const float* queries, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters) {
    return guard([&] {
        if (e && !e->d_peer_xchg) fail(SINKR_INVALID_ARGUMENT, "peer merge not set up (sinkr_peer_open)");
        if (e && e->peer_poisoned)
            fail(SINKR_LOGIC_ERROR, "peer merge disabled after a watchdog timeout (set it up again)");
        decode_host(e, queries, layer, config, options, outputs, groups, head_scores, counters, 3);
    });
}

static void decode_host(sinkr_engine* e, const float* queries, size_t layer,
                        const sinkr_routing_config* config, const sinkr_engine_options* options,
                        float* outputs, sinkr_group_info* groups, double* head_scores,
                        sinkr_load_counters* counters, int mode) {
    {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        if (!queries) fail(SINKR_INVALID_ARGUMENT, "queries span must be H_q x D for one layer");
        CK(cudaSetDevice(e->device));
        stage_params(e, layer, config, options, true);  // validates before touching q
        const size_t qbytes = e->B * e->cfg.num_q_heads * e->D * 4;
        // params were written into h_in by stage_params; append the queries
        // (unless the caller filled the pinned query area itself) and upload
        // the whole input block in one H2D copy.
        if (queries != reinterpret_cast<const float*>(e->h_in + e->off_q))
            std::memcpy(e->h_in + e->off_q, queries, qbytes);
        if (e->fused && !e->timing && io_mode() != 0) {
            run_io_graph(e, mode);  // H2D + step kernel, results land in mapped h_res
            finish_io(e);
        } else {
            CK(cudaMemcpyAsync(e->d_in, e->h_in, e->in_bytes, cudaMemcpyHostToDevice, e->stream));
            CK(cudaEventRecord(e->ev_in, e->stream));
            e->ev_in_pending = true;
            float* d_out = reinterpret_cast<float*>(e->d_res);
            run_graph(e, reinterpret_cast<const float*>(e->d_in + e->off_q), d_out, mode);
            CK(cudaMemcpyAsync(e->h_res, e->d_res, e->res_bytes, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
        }
        if (!e->fused) {
            dev::WorkState ws;
            CK(cudaMemcpy(&ws, e->d_ws, sizeof(ws), cudaMemcpyDeviceToHost));
            if (ws.error) fail(SINKR_RUNTIME_ERROR, "decode partial-slot overflow");
        }
        if (outputs && outputs != reinterpret_cast<float*>(e->h_res)) std::memcpy(outputs, e->h_res, qbytes);
        fill_info(e, layer, config, groups, head_scores, counters, options);
    }
}

// ---- per-token KV append (kv_cache.cpp:61-84) ---------------------
// The decode loop's append of the new token to every (seq, kv_head) slot of a
// layer, stream-ordered on the engine stream: one small kernel, no host sync
// (first rows of empty slots take the synchronous host path, which captures
// the anchor and checks it like KvCache::append).
sinkr_status sinkr_kv_append_token_async(sinkr_engine* e, size_t layer, const float* d_k_new,
                                         const float* d_v_new) {
    return guard([&] {
        if (!e || !d_k_new || !d_v_new) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        if (check_token_append(e, layer)) {
            const size_t H = e->cfg.num_kv_heads;
            for (size_t u = 0; u < e->U; ++u) {
                const sinkr_status st = sinkr_kv_append_device_f32(e, u / H, layer, u % H, d_k_new + u * e->D,
                                                                   d_v_new + u * e->D, 1);
                if (st != SINKR_OK) fail(st, g_err);
            }
            return;
        }
        sync_dlen(e);
        launch_append(e, layer, d_k_new, d_v_new);
        for (size_t u = 0; u < e->U; ++u) ++e->len[layer * e->U + u];
    });
}

// One decode step of `layer` that first appends the new token (host rows
// k_new / v_new [B][H_kv][D] f32) to every slot of the layer and then runs the
// routed step over the grown cache (the reference's append-then-step,
// a Sink group skips the new row too).  One graph per call: H2D
// of params + queries + new rows, the append kernel, the step kernel writing
// zero-copy into pinned host memory.  As in the reference, the sequence's
// slots must be uniform after the append (token_count, kv_cache.cpp:90-96).
sinkr_status sinkr_decode_append_step(sinkr_engine* e, const float* queries, const float* k_new,
                                      const float* v_new, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        if (!queries) fail(SINKR_INVALID_ARGUMENT, "queries span must be H_q x D for one layer");
        if (!k_new || !v_new) fail(SINKR_INVALID_ARGUMENT, "k/v row size does not match head_dim");
        if (!config) fail(SINKR_INVALID_ARGUMENT, "routing config is null");
        CK(cudaSetDevice(e->device));
        const size_t H = e->cfg.num_kv_heads, D = e->D;
        if (check_token_append(e, layer)) {  // first rows: the host append path
            for (size_t u = 0; u < e->U; ++u) {
                const sinkr_status st = sinkr_kv_append(e, u / H, layer, u % H, k_new + u * D, v_new + u * D, 1);
                if (st != SINKR_OK) fail(st, g_err);
            }
            decode_host(e, queries, layer, config, options, outputs, groups, head_scores, counters, 0);
            return;
        }
        // every slot of each sequence must be uniform once this layer grows
        for (size_t s = 0; s < e->B; ++s) {
            const size_t n = e->len[e->slot_index(layer, s, 0)] + 1;
            for (size_t l = 0; l < e->layers; ++l)
                for (size_t g = 0; g < H; ++g)
                    if (e->len[e->slot_index(l, s, g)] + (l == layer ? 1 : 0) != n)
                        fail(SINKR_LOGIC_ERROR, "kv cache lengths are ragged across slots");
        }
        sync_dlen(e);  // the kernel appends at the device lengths (pre-append)
        for (size_t u = 0; u < e->U; ++u) ++e->len[layer * e->U + u];
        stage_params(e, layer, config, options, true);
        const size_t qbytes = e->B * e->cfg.num_q_heads * D * 4;
        std::memcpy(e->h_in + e->off_q, queries, qbytes);
        std::memcpy(e->h_in + e->off_kvn, k_new, e->U * D * 4);
        std::memcpy(e->h_in + e->off_kvn + e->U * D * 4, v_new, e->U * D * 4);
        if (e->fused && !e->timing && io_mode() != 0) {
            run_io_graph(e, 0, (long)layer);
            finish_io(e);
        } else {
            CK(cudaMemcpyAsync(e->d_in, e->h_in, e->in_bytes_append, cudaMemcpyHostToDevice, e->stream));
            CK(cudaEventRecord(e->ev_in, e->stream));
            e->ev_in_pending = true;
            const float* kn = reinterpret_cast<const float*>(e->d_in + e->off_kvn);
            launch_append(e, layer, kn, kn + e->U * D);
            run_graph(e, reinterpret_cast<const float*>(e->d_in + e->off_q), reinterpret_cast<float*>(e->d_res), 0);
            e->last_launches += 1;
            CK(cudaMemcpyAsync(e->h_res, e->d_res, e->res_bytes, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
        }
        if (outputs && outputs != reinterpret_cast<float*>(e->h_res)) std::memcpy(outputs, e->h_res, qbytes);
        fill_info(e, layer, config, groups, head_scores, counters, options);
    });
}

// splitk_attention (attention.cpp:204-235) of ONE cached group on the GPU:
// the fused step kernel with the route forced (ProbeParams.only_unit), so the
// group streams exactly like an Active group of a routed step and every other
// group is skipped.  The split count is validated like split_ranges
// (attention.cpp:185-190); the GPU picks its own split.
sinkr_status sinkr_group_attention(sinkr_engine* e, const float* group_queries, size_t seq,
                                   size_t layer, size_t kv_head, size_t num_splits, float* out,
                                   sinkr_load_counters* counters) {
    return guard([&] {
        if (!e || !group_queries || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        check_slot(e, seq, layer, kv_head);
        const size_t L = e->len[e->slot_index(layer, seq, kv_head)];
        if (L == 0) fail(SINKR_INVALID_ARGUMENT, "attention needs at least one token");
        if (num_splits == 0 || num_splits > L)
            fail(SINKR_INVALID_ARGUMENT, "num_splits must be in [1, len], got " +
                                             std::to_string(num_splits) + " for len " +
                                             std::to_string(L));
        const size_t H = e->cfg.num_kv_heads, Hq = e->cfg.num_q_heads, r = e->r, D = e->D;
        const size_t u = seq * H + kv_head, row0 = (seq * Hq + kv_head * r) * D;
        wait_input_block(e);
        auto* hdr = reinterpret_cast<dev::StepHdr*>(e->h_in);
        auto* tau = reinterpret_cast<double*>(e->h_in + e->off_tau);
        auto* len = reinterpret_cast<uint32_t*>(e->h_in + e->off_len);
        hdr->layer = (uint32_t)layer;
        hdr->flags = 0;
        hdr->pad[0] = hdr->pad[1] = 0;
        for (size_t s = 0; s < e->B; ++s) {
            tau[s] = 2.0;  // (no decision is taken from it)
            len[s] = s == seq ? (uint32_t)L : 0u;
        }
        std::memset(&e->pp, 0, sizeof(e->pp));
        e->pp.layer = (uint32_t)layer;
        e->pp.inline_seqs = e->B <= (size_t)dev::kParamSeqs ? 1u : 0u;
        if (e->pp.inline_seqs)
            for (size_t s = 0; s < e->B; ++s) {
                e->pp.tau[s] = tau[s];
                e->pp.len[s] = len[s];
            }
        e->pp.only_unit = (uint32_t)(u + 1);
        e->params_valid = false;  // the next routed step uploads its own params
        float* q = reinterpret_cast<float*>(e->h_in + e->off_q);
        std::memset(q, 0, e->B * Hq * D * 4);
        std::memcpy(q + row0, group_queries, r * D * 4);
        if (e->fused && !e->timing && io_mode() != 0) {
            run_io_graph(e);
            finish_io(e);
        } else {
            CK(cudaMemcpyAsync(e->d_in, e->h_in, e->in_bytes, cudaMemcpyHostToDevice, e->stream));
            CK(cudaEventRecord(e->ev_in, e->stream));
            e->ev_in_pending = true;
            run_graph(e, reinterpret_cast<const float*>(e->d_in + e->off_q),
                      reinterpret_cast<float*>(e->d_res), 0);
            CK(cudaMemcpyAsync(e->h_res, e->d_res, e->res_bytes, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
        }
        e->pp.only_unit = 0;
        const auto* fl = reinterpret_cast<const uint32_t*>(e->h_res + e->off_fl);
        const auto* tok = reinterpret_cast<const unsigned long long*>(e->h_res + e->off_tok);
        if (!(fl[u] & dev::kActive) || tok[u] != L)
            fail(SINKR_RUNTIME_ERROR, "group attention: the forced group was not streamed");
        std::memcpy(out, reinterpret_cast<const float*>(e->h_res) + row0, r * D * 4);
        if (counters) {
            *counters = sinkr_load_counters{};
            counters->kv_floats_loaded = 2ull * L * D;  // attention.cpp:219
        }
    });
}

// attend_chunk (attention.cpp:101-142) of one group's r query heads over the
// cached rows [from, to) of (seq, layer, kv_head) -- the reference's
// run_task pairing of KvCache::historical (kv_cache.cpp:106-121) with
// attend_chunk (router.cpp:149-160) -- returning the chunk's SplitPartial
// (fp64 m[r], l[r], acc[r][D]; tokens = to - from).  The span kernel
// (span.cuh) reads the bf16 rows in place on the engine stream.
sinkr_status sinkr_attend_chunk_cached(sinkr_engine* e, const float* group_queries, size_t seq,
                                       size_t layer, size_t kv_head, size_t from, size_t to,
                                       size_t block_size, double* m, double* l, double* acc,
                                       uint64_t* tokens) {
    return guard([&] {
        if (!e || !group_queries || !m || !l || !acc) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        check_slot(e, seq, layer, kv_head);
        const size_t idx = e->slot_index(layer, seq, kv_head), D = e->D, r = e->r;
        if (from > to || to > e->len[idx])
            fail(SINKR_OUT_OF_RANGE, "historical range [" + std::to_string(from) + ", " +
                                         std::to_string(to) + ") exceeds length " +
                                         std::to_string(e->len[idx]));
        if (to == from) fail(SINKR_INVALID_ARGUMENT, "attention needs at least one token");
        if (block_size == 0) fail(SINKR_INVALID_ARGUMENT, "block_size must be positive");
        const size_t len = to - from;
        const size_t qb = align_up(r * D * 4, 256), pb = align_up(r * (D + 2) * 8, 256);
        const size_t need = qb + pb + span::attend_scratch_bytes(r, D, len, e->num_sms);
        if (e->span_bytes < need) {
            CK(cudaStreamSynchronize(e->stream));
            cudaFree(e->d_span);
            e->d_span = nullptr;
            e->span_bytes = 0;
            CK(cudaMalloc(&e->d_span, need));
            e->span_bytes = need;
        }
        float* d_q = reinterpret_cast<float*>(e->d_span);
        double* d_m = reinterpret_cast<double*>(e->d_span + qb);
        double* d_l = d_m + r;
        double* d_acc = d_l + r;
        CK(cudaMemcpyAsync(d_q, group_queries, r * D * 4, cudaMemcpyHostToDevice, e->stream));
        const size_t off = (e->row_base(layer, seq, kv_head) + from) * D;
        span::attend_device(e->stream, d_q, r, D, e->d_k + off, e->d_v + off, len, e->d_span + qb + pb,
                            d_m, d_l, d_acc, e->num_sms);
        CK(cudaMemcpyAsync(m, d_m, r * 8, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaMemcpyAsync(l, d_l, r * 8, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaMemcpyAsync(acc, d_acc, r * D * 8, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
        if (tokens) *tokens = len;
    });
}

sinkr_status sinkr_routed_decode_step(sinkr_engine* e, const float* queries, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters) {
    if (e && e->B != 1) {
        g_err = "sinkr_routed_decode_step serves single-sequence engines; use _batch";
        return SINKR_INVALID_ARGUMENT;
    }
    return sinkr_routed_decode_batch(e, queries, layer, config, options, outputs, groups,
                                     head_scores, counters);
}

sinkr_status sinkr_routed_decode_async(sinkr_engine* e, const float* d_queries, size_t layer,
                                       const sinkr_routing_config* config,
                                       const sinkr_engine_options* options, float* d_outputs) {
    return guard([&] {
        if (!e || !d_queries || !d_outputs) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        stage_params(e, layer, config, options, false);
        run_graph(e, d_queries, d_outputs, 0);
    });
}

sinkr_status sinkr_fetch_step_info(sinkr_engine* e, sinkr_group_info* groups,
                                   double* head_scores, sinkr_load_counters* counters) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        CK(cudaMemcpyAsync(e->h_res + e->off_hs, e->d_res + e->off_hs, e->res_bytes - e->off_hs,
                           cudaMemcpyDeviceToHost, e->stream));
        if (e->fused)
            CK(cudaStreamSynchronize(e->stream));
        else
            check_error_flag(e);
        const auto* hdr = reinterpret_cast<const dev::StepHdr*>(e->h_in);
        fill_info(e, hdr->layer, nullptr, groups, head_scores, counters, nullptr);
    });
}

// Score-collection mode (calibration.hpp:74-76): the routing
// phase alone — the probe kernel scores every head and group and records the
// decisions, no K/V row is streamed.  Calibration populations therefore cost
// one small launch per sample instead of a full decode step.
sinkr_status sinkr_collect_scores(sinkr_engine* e, const float* queries, size_t layer,
                                  const sinkr_routing_config* config, double* head_scores,
                                  double* group_scores, int32_t* sink) {
    return guard([&] {
        if (!e || !queries) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        sinkr_routing_config none{};
        none.profile.coeffs[3] = 2.0;  // ThresholdProfile::constant(2.0): nothing sinks
        none.profile.length_normalizer = 1.0;
        none.profile.clamp_lo = 0.0;
        none.profile.clamp_hi = 2.0;
        stage_params(e, layer, config ? config : &none, nullptr, true);
        const size_t NH = e->B * e->cfg.num_q_heads;
        std::memcpy(e->h_in + e->off_q, queries, NH * e->D * 4);
        dev::DevTables t = e->tables(reinterpret_cast<const float*>(e->d_in + e->off_q));
        // scores and flags straight into the mapped result block (as the step
        // path does): no D2H copy in the call
        const bool zc = io_mode() == 1 && e->h_res_dev;
        if (zc) {
            t.head_scores = reinterpret_cast<double*>(e->h_res_dev + e->off_hs);
            t.group_scores = reinterpret_cast<double*>(e->h_res_dev + e->off_gs);
            t.unit_flags = reinterpret_cast<uint32_t*>(e->h_res_dev + e->off_fl);
            t.tokens = reinterpret_cast<unsigned long long*>(e->h_res_dev + e->off_tok);
            t.done = e->h_done_dev;  // the probe's last CTA sets it after its writes
        }
        auto enqueue = [&] {
            if (zc)
                launch_upload(e, e->in_bytes);  // graph node: the upload kernel (see launch_upload)
            else
                CK(cudaMemcpyAsync(e->d_in, e->h_in, e->in_bytes, cudaMemcpyHostToDevice, e->stream));
            switch (e->D) {
                case 32: dev::probe_kernel<32><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
                case 64: dev::probe_kernel<64><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
                default: dev::probe_kernel<128><<<e->probe_grid, dev::kProbeThreads, probe_smem(e), e->stream>>>(t, e->pp); break;
            }
            CK(cudaGetLastError());
        };
        if (zc) {
            // one graph (upload + probe), captured once per engine; the probe's
            // by-value parameters are patched when they change
            const auto key = std::make_tuple((const void*)e->h_in, (void*)e->h_res, 4);
            auto it = e->graphs.find(key);
            if (it == e->graphs.end()) {
                sinkr_engine::GraphEntry ge;
                CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
                try {
                    enqueue();
                } catch (...) {
                    cudaStreamEndCapture(e->stream, &ge.graph);
                    if (ge.graph) cudaGraphDestroy(ge.graph);
                    throw;
                }
                CK(cudaStreamEndCapture(e->stream, &ge.graph));
                CK(cudaGraphInstantiate(&ge.exec, ge.graph, 0));
                size_t n = 0;
                CK(cudaGraphGetNodes(ge.graph, nullptr, &n));
                std::vector<cudaGraphNode_t> nodes(n);
                CK(cudaGraphGetNodes(ge.graph, nodes.data(), &n));
                const void* probe_fn = e->D == 32 ? (const void*)dev::probe_kernel<32>
                                       : e->D == 64 ? (const void*)dev::probe_kernel<64>
                                                    : (const void*)dev::probe_kernel<128>;
                for (auto nd : nodes) {
                    cudaGraphNodeType ty;
                    CK(cudaGraphNodeGetType(nd, &ty));
                    if (ty != cudaGraphNodeTypeKernel) continue;
                    cudaKernelNodeParams kp{};
                    CK(cudaGraphKernelNodeGetParams(nd, &kp));
                    if (kp.func != probe_fn) continue;
                    ge.probe_kp = kp;
                    ge.probe = nd;
                }
                if (!ge.probe) fail(SINKR_CUDA_ERROR, "probe node not found in the captured graph");
                ge.probe_t = t;
                ge.pp = e->pp;
                it = e->graphs.emplace(key, ge).first;
            }
            auto& ge = it->second;
            if (std::memcmp(&ge.pp, &e->pp, sizeof(e->pp)) != 0) {
                ge.pp = e->pp;
                void* args[2] = {&ge.probe_t, &ge.pp};
                cudaKernelNodeParams kp = ge.probe_kp;
                kp.kernelParams = args;
                kp.extra = nullptr;
                CK(cudaGraphExecKernelNodeSetParams(ge.exec, ge.probe, &kp));
            }
            *reinterpret_cast<volatile uint32_t*>(e->h_done) = 0u;
            CK(cudaGraphLaunch(ge.exec, e->stream));
            finish_io(e);  // spins on the completion word
        } else {
            enqueue();
            // head scores, group scores and flags are contiguous in the result block
            CK(cudaMemcpyAsync(e->h_res + e->off_hs, e->d_res + e->off_hs, e->off_status - e->off_hs,
                               cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
        }
        const auto* hs = reinterpret_cast<const double*>(e->h_res + e->off_hs);
        const auto* gs = reinterpret_cast<const double*>(e->h_res + e->off_gs);
        const auto* fl = reinterpret_cast<const uint32_t*>(e->h_res + e->off_fl);
        if (head_scores) std::memcpy(head_scores, hs, NH * sizeof(double));
        if (group_scores) std::memcpy(group_scores, gs, e->U * sizeof(double));
        if (sink)
            for (size_t u = 0; u < e->U; ++u) sink[u] = (config && (fl[u] & dev::kSink)) ? 1 : 0;
    });
}

sinkr_status sinkr_collect_scores_batch(sinkr_engine* e, const float* queries, size_t n_samples,
                                        size_t layer, const sinkr_routing_config* config,
                                        double* head_scores, double* group_scores, int32_t* sink) {
    return guard([&] {
        if (!e || !queries) fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (layer >= e->layers) fail(SINKR_OUT_OF_RANGE, "layer index out of range");
        if (n_samples == 0) return;
        CK(cudaSetDevice(e->device));
        const size_t NH = e->B * e->cfg.num_q_heads, U = e->U, D = e->D;
        for (size_t s = 0; s < e->B; ++s)
            for (size_t g = 0; g < e->cfg.num_kv_heads; ++g)
                if (!e->anchored[e->slot_index(layer, s, g)])
                    fail(SINKR_RUNTIME_ERROR, "anchor requested from empty cache slot");
        if (n_samples * U > (size_t)0xFFFFFFFFu / 2) fail(SINKR_INVALID_ARGUMENT, "too many samples");
        // device scratch: tau [B] | queries [n][NH][D] | head [n][NH] | group [n][U] | sink [n][U]
        const size_t off_q = align_up(e->B * 8, 256);
        const size_t off_h = align_up(off_q + n_samples * NH * D * 4, 256);
        const size_t off_g = align_up(off_h + n_samples * NH * 8, 256);
        const size_t off_s = align_up(off_g + n_samples * U * 8, 256);
        const size_t bytes = off_s + n_samples * U * 4;
        if (bytes > e->score_scratch_bytes) {
            if (e->d_score_scratch) CK(cudaFree(e->d_score_scratch));
            e->d_score_scratch = nullptr;
            e->score_scratch_bytes = 0;
            CK(cudaMalloc(&e->d_score_scratch, bytes));
            e->score_scratch_bytes = bytes;
        }
        uint8_t* d = e->d_score_scratch;
        std::vector<double> tau(e->B, 0.0);
        dev::ScoreBatchArgs a{};
        if (config) {
            for (size_t s = 0; s < e->B; ++s) {
                const size_t L = token_count(e, s);
                if (L == 0) fail(SINKR_RUNTIME_ERROR, "routed decode over an empty cache");
                tau[s] = threshold_for_length(L, config->profile);
            }
            a.flags = (config->sink_on_tie ? dev::kSinkOnTie : 0u) |
                      (layer_excluded(layer, *config) ? dev::kLayerExcluded : 0u);
            a.has_cfg = 1;
        }
        CK(cudaMemcpyAsync(d, tau.data(), e->B * 8, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(d + off_q, queries, n_samples * NH * D * 4, cudaMemcpyHostToDevice, e->stream));
        a.q = reinterpret_cast<const float*>(d + off_q);
        a.anchors = e->d_anchor + layer * U * D;
        a.anchor_norm = e->d_anchor_norm + layer * U;
        a.tau = reinterpret_cast<const double*>(d);
        a.head_scores = reinterpret_cast<double*>(d + off_h);
        a.group_scores = reinterpret_cast<double*>(d + off_g);
        a.sink = reinterpret_cast<int32_t*>(d + off_s);
        a.n = (uint32_t)n_samples;
        a.U = (uint32_t)U;
        a.Hkv = (uint32_t)e->cfg.num_kv_heads;
        a.r = (uint32_t)e->r;
        a.units_per_cta = (uint32_t)std::max<size_t>(1, dev::kScoreHeads / e->r);
        const unsigned grid = (unsigned)((n_samples * U + a.units_per_cta - 1) / a.units_per_cta);
        const size_t smem = 2 * dev::kScoreHeads * (D + 1) * 8;
        switch (D) {
            case 32: dev::score_batch_kernel<32><<<grid, dev::kScoreThreads, smem, e->stream>>>(a); break;
            case 64: dev::score_batch_kernel<64><<<grid, dev::kScoreThreads, smem, e->stream>>>(a); break;
            default: dev::score_batch_kernel<128><<<grid, dev::kScoreThreads, smem, e->stream>>>(a); break;
        }
        CK(cudaGetLastError());
        if (head_scores)
            CK(cudaMemcpyAsync(head_scores, d + off_h, n_samples * NH * 8, cudaMemcpyDeviceToHost, e->stream));
        if (group_scores)
            CK(cudaMemcpyAsync(group_scores, d + off_g, n_samples * U * 8, cudaMemcpyDeviceToHost, e->stream));
        if (sink) CK(cudaMemcpyAsync(sink, d + off_s, n_samples * U * 4, cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
    });
}

static void launch_bos(sinkr_engine* e, const dev::BosArgs& a) {
#define SINKR_BOS_LAUNCH(DD)                                                                      \
    {                                                                                             \
        constexpr int smem = dev::BosCfg<DD>::kSmemBytes; /* attribute set at creation */      \
        if (e->wide)                                                                              \
            dev::bos_stream_kernel<DD, 2><<<a.G, dev::kBosThreads, smem, e->stream>>>(e->tmk, a); \
        else                                                                                      \
            dev::bos_stream_kernel<DD, 1><<<a.G, dev::kBosThreads, smem, e->stream>>>(e->tmk, a); \
    }
    switch (e->D) {
        case 32: SINKR_BOS_LAUNCH(32) break;
        case 64: SINKR_BOS_LAUNCH(64) break;
        default: SINKR_BOS_LAUNCH(128) break;
    }
#undef SINKR_BOS_LAUNCH
}

// Full-attention BOS mass (analysis.cuh).  Queries are staged in the input
// block's query area; the scratch persists in the engine, grown on demand.
static void run_bos(sinkr_engine* e, const float* queries, size_t q_floats, size_t q_offset,
                    size_t layer, uint32_t u_first, uint32_t n_units, double* alpha0,
                    float* weights) {
    if (layer >= e->layers) fail(SINKR_OUT_OF_RANGE, "layer index out of range");
    const size_t U = e->U, r = e->r, D = e->D;
    std::vector<uint32_t> pre(n_units + 1, 0);
    for (uint32_t i = 0; i < n_units; ++i) {
        const size_t L = e->len[layer * U + u_first + i];
        if (L == 0) fail(SINKR_RUNTIME_ERROR, "attention over an empty cache slot");
        pre[i + 1] = pre[i] + (uint32_t)L;
    }
    const uint32_t T = pre[n_units];
    // one stream CTA per SM (the ring takes ~128 KB), >= one stage of tokens each
    const uint32_t G = std::max<uint32_t>(
        1, std::min<uint32_t>((uint32_t)e->num_sms, (T + dev::kBosTok - 1) / dev::kBosTok));
    // scratch: ctr[2][1+U] (zeroed at allocation; each call's finish zeroes the other set) | pre[n+1] |
    //          part[n][G][r][2] | z0[U*r] | stats[U*r][2] | logits | weights (alpha0: mapped h_bos)
    const size_t off_pre = align_up(2 * (1 + U) * 4, 256);
    const size_t off_part = align_up(off_pre + (n_units + 1) * 4, 256);
    const size_t off_z0 = align_up(off_part + (size_t)n_units * G * r * 2 * 4, 256);
    const size_t off_st = align_up(off_z0 + U * r * 4, 256);
    const size_t off_z = align_up(off_st + U * r * 2 * 4, 256);
    const size_t wbytes = weights ? r * (size_t)T * 4 : 0;
    const size_t off_w = align_up(off_z + wbytes, 256);
    const size_t need = off_w + wbytes;
    if (e->bos_bytes < need) {
        CK(cudaStreamSynchronize(e->stream));
        e->drop_bos_graphs();
        cudaFree(e->d_bos);
        e->d_bos = nullptr;
        e->bos_bytes = 0;
        CK(cudaMalloc(&e->d_bos, need));
        CK(cudaMemsetAsync(e->d_bos, 0, 2 * (1 + U) * 4, e->stream));
        e->bos_parity = 0;
        e->bos_bytes = need;
    }
    uint8_t* scratch = e->d_bos;
    const uint32_t nh = n_units * (uint32_t)r;
    // pinned + mapped: prefix up by copy, alpha0 [U*r] written by the finish
    // kernel straight into host memory
    const size_t h_a0 = align_up((n_units + 1) * 4, 64), h_need = h_a0 + U * r * 8;
    if (e->h_bos_bytes < h_need) {
        CK(cudaStreamSynchronize(e->stream));
        e->drop_bos_graphs();
        if (e->h_bos) cudaFreeHost(e->h_bos);
        e->h_bos = nullptr;
        e->h_bos_bytes = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&e->h_bos), h_need, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_bos_dev), e->h_bos, 0));
        e->h_bos_bytes = h_need;
    }
    wait_input_block(e);  // the input block is free
    std::memcpy(e->h_in + e->off_q + q_offset * 4, queries, q_floats * 4);
    std::memcpy(e->h_bos, pre.data(), (n_units + 1) * 4);
    const uint32_t parity = e->bos_parity;
    dev::BosArgs a{};
    a.pre = reinterpret_cast<const uint32_t*>(scratch + off_pre);
    a.q = reinterpret_cast<const float*>(e->d_in + e->off_q);
    a.part = reinterpret_cast<float*>(scratch + off_part);
    a.ctr = reinterpret_cast<uint32_t*>(scratch) + e->bos_parity * (1 + U);
    a.ctr_next = reinterpret_cast<uint32_t*>(scratch) + (1 - e->bos_parity) * (1 + U);
    a.ctr_len = (uint32_t)(1 + U);
    e->bos_parity ^= 1u;
    a.z0 = reinterpret_cast<float*>(scratch + off_z0);
    a.stats = reinterpret_cast<float*>(scratch + off_st);
    a.alpha0 = reinterpret_cast<double*>(e->h_bos_dev + h_a0);
    a.zout = weights ? reinterpret_cast<float*>(scratch + off_z) : nullptr;
    a.weights = reinterpret_cast<float*>(scratch + off_w);
    a.r = (uint32_t)r;
    a.cap = (uint32_t)e->cap;
    a.slot0 = (uint32_t)(layer * U);
    a.u_first = u_first;
    a.n_units = n_units;
    a.G = G;
    a.qscale = (1.0f / std::sqrt((float)D)) * 1.4426950408889634f;
    // from here the counter sets are in flight: if anything fails before the
    // finish kernel has zeroed the next set, the scratch is dropped (the next
    // call reallocates and zeroes it)
    struct DropScratchOnError {
        sinkr_engine* e;
        bool armed = true;
        ~DropScratchOnError() {
            if (!armed) return;
            cudaStreamSynchronize(e->stream);
            e->drop_bos_graphs();
            cudaFree(e->d_bos);
            e->d_bos = nullptr;
            e->bos_bytes = 0;
        }
    } guard_scratch{e};
    static_assert(dev::kBosHeads >= dev::kMaxRWide, "one stream pass covers a GQA group");
    // uploads (query rows, token prefix) + stream + finish [+ weights]: one graph
    auto enqueue = [&] {
        CK(cudaMemcpyAsync(e->d_in + e->off_q + q_offset * 4, e->h_in + e->off_q + q_offset * 4,
                           q_floats * 4, cudaMemcpyHostToDevice, e->stream));
        CK(cudaMemcpyAsync(scratch + off_pre, e->h_bos, (n_units + 1) * 4, cudaMemcpyHostToDevice,
                           e->stream));
        // event-record nodes inside the graph: device time of the kernels alone
        CK(cudaEventRecordWithFlags(e->ev_bos[0], e->stream, cudaEventRecordExternal));
        launch_bos(e, a);
        dev::bos_finish_kernel<<<std::max<uint32_t>(1, (nh + 7) / 8), 256, 0, e->stream>>>(a);
        if (weights) {
            const uint32_t blocks = std::min<uint32_t>((uint32_t)((r * (size_t)T + 255) / 256),
                                                       8u * (uint32_t)e->num_sms);
            dev::weights_kernel<<<blocks, 256, 0, e->stream>>>(a);
        }
        CK(cudaGetLastError());
        CK(cudaEventRecordWithFlags(e->ev_bos[1], e->stream, cudaEventRecordExternal));
    };
    // T is part of the key: the captured kernel arguments (a.weights =
    // scratch + off_w, the weights grid) move with the token count even when
    // the scratch is not reallocated
    const std::array<uint64_t, 7> key = {layer, u_first, n_units, G, weights ? 1u : 0u, parity, T};
    auto it = e->bos_graphs.find(key);
    if (it == e->bos_graphs.end()) {
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue();
        } catch (...) {
            cudaStreamEndCapture(e->stream, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CK(cudaStreamEndCapture(e->stream, &g));
        cudaGraphExec_t x = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&x, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
        it = e->bos_graphs.emplace(key, x).first;
    }
    CK(cudaGraphLaunch(it->second, e->stream));
    if (weights)
        CK(cudaMemcpyAsync(weights, scratch + off_w, wbytes, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    guard_scratch.armed = false;
    std::memcpy(alpha0, e->h_bos + h_a0 + (size_t)u_first * r * 8, (size_t)nh * 8);
    CK(cudaEventElapsedTime(&e->bos_ms, e->ev_bos[0], e->ev_bos[1]));
}

sinkr_status sinkr_attention_last_kernel_seconds(sinkr_engine* e, double* seconds) {
    return guard([&] {
        if (!e || !seconds) fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (e->bos_ms < 0.f) fail(SINKR_RUNTIME_ERROR, "no analysis pass has run on this engine");
        *seconds = e->bos_ms * 1e-3;
    });
}

sinkr_status sinkr_attention_bos_mass(sinkr_engine* e, const float* queries, size_t layer,
                                      double* alpha0) {
    return guard([&] {
        if (!e || !queries || !alpha0) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        const size_t nq = e->B * e->cfg.num_q_heads * e->D;
        run_bos(e, queries, nq, 0, layer, 0, (uint32_t)e->U, alpha0, nullptr);
    });
}

sinkr_status sinkr_attention_weights(sinkr_engine* e, const float* queries, size_t seq,
                                     size_t layer, size_t kv_head, float* weights) {
    return guard([&] {
        if (!e || !queries || !weights) fail(SINKR_INVALID_ARGUMENT, "null argument");
        check_slot(e, seq, layer, kv_head);
        CK(cudaSetDevice(e->device));
        const uint32_t u = (uint32_t)(seq * e->cfg.num_kv_heads + kv_head);
        std::vector<double> a0(e->r);
        run_bos(e, queries, e->r * e->D, (size_t)u * e->r * e->D, layer, u, 1, a0.data(), weights);
    });
}

size_t sinkr_rank_partial_floats(sinkr_engine* e) { return e ? e->U * e->PS : 0; }

sinkr_status sinkr_decode_rank_partial_async(sinkr_engine* e, const float* d_queries,
                                             size_t layer, const sinkr_routing_config* config,
                                             const sinkr_engine_options* options,
                                             float* d_partial) {
    return guard([&] {
        if (!e || !d_queries || !d_partial) fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        stage_params(e, layer, config, options, false);
        run_graph(e, d_queries, d_partial, 1);
    });
}

sinkr_status sinkr_merge_rank_partials_async(sinkr_engine* e, const float* d_gathered,
                                             size_t num_ranks, float* d_outputs) {
    return guard([&] {
        if (!e || !d_gathered || !d_outputs || num_ranks == 0)
            fail(SINKR_INVALID_ARGUMENT, "null argument");
        CK(cudaSetDevice(e->device));
        const dev::DevTables t = e->tables(nullptr);
        launch_combine(e, t, d_gathered, e->PS, e->U * e->PS, (uint32_t)num_ranks, d_outputs, 0,
                       num_ranks);
        CK(cudaGetLastError());
    });
}

// ---- fused sequence-sharded merge over peer memory (mode 3) ------------------
static void peer_tables(sinkr_engine* e, const std::vector<uint8_t*>& blocks) {
    std::vector<unsigned long long*> px(e->world);
    for (uint32_t q = 0; q < e->world; ++q) px[q] = reinterpret_cast<unsigned long long*>(blocks[q]);
    if (!e->d_peer_xchg) CK(cudaMalloc(&e->d_peer_xchg, 8 * sizeof(unsigned long long*)));
    CK(cudaMemcpy(e->d_peer_xchg, px.data(), e->world * sizeof(unsigned long long*), cudaMemcpyHostToDevice));
}

sinkr_status sinkr_peer_setup(sinkr_engine* e, uint32_t world, uint32_t rank, size_t* block_bytes) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        if (world == 0 || world > 8 || rank >= world)
            fail(SINKR_INVALID_ARGUMENT, "peer merge needs 1 <= world <= 8 and rank < world");
        if (!e->fused) fail(SINKR_INVALID_ARGUMENT, "peer merge needs the fused step kernel");
        CK(cudaSetDevice(e->device));
        if (e->d_xchg) {
            // set up again (after a watchdog timeout every rank must): a
            // fresh, zeroed exchange block and step tags from zero, so no
            // word of an earlier step can carry a valid tag; every rank then
            // connects again
            CK(cudaStreamSynchronize(e->stream));
            for (auto& kv : e->graphs) {
                cudaGraphExecDestroy(kv.second.exec);
                cudaGraphDestroy(kv.second.graph);
            }
            e->graphs.clear();
            for (void* pb : e->ipc_opened) cudaIpcCloseMemHandle(pb);
            e->ipc_opened.clear();
            cudaFree(e->d_xchg);
            cudaFree(e->d_peer_xchg);
            e->d_xchg = nullptr;
            e->d_peer_xchg = nullptr;
            CK(cudaMemset(e->d_cta_epoch + e->grid, 0, e->grid * 4));  // mode-3 step counts
            e->peer_poisoned = false;
        }
        e->world = world;
        e->rank = rank;
        // [2 parities][world][U][r(D+2)] LL words (8 B each)
        e->xchg_words = 2ull * world * e->U * e->PS;
        e->xchg_bytes = align_up(e->xchg_words * 8, 256);
        CK(cudaMalloc(&e->d_xchg, e->xchg_bytes));
        CK(cudaMemset(e->d_xchg, 0, e->xchg_bytes));
        if (block_bytes) *block_bytes = e->xchg_bytes;
    });
}

sinkr_status sinkr_peer_ipc_handle(sinkr_engine* e, void* handle) {
    return guard([&] {
        if (!e || !handle || !e->d_xchg) fail(SINKR_INVALID_ARGUMENT, "peer merge not set up");
        CK(cudaSetDevice(e->device));
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, e->d_xchg));
        std::memcpy(handle, &h, sizeof(h));
    });
}

sinkr_status sinkr_peer_open(sinkr_engine* e, const void* handles) {
    return guard([&] {
        if (!e || !handles || !e->d_xchg) fail(SINKR_INVALID_ARGUMENT, "peer merge not set up");
        CK(cudaSetDevice(e->device));
        std::vector<uint8_t*> blocks(e->world);
        for (uint32_t q = 0; q < e->world; ++q) {
            if (q == e->rank) {
                blocks[q] = e->d_xchg;
                continue;
            }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const uint8_t*>(handles) + q * sizeof(h), sizeof(h));
            void* ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
            e->ipc_opened.push_back(ptr);
            blocks[q] = static_cast<uint8_t*>(ptr);
        }
        peer_tables(e, blocks);
    });
}

sinkr_status sinkr_peer_set_blocks(sinkr_engine* e, void* const* blocks) {
    return guard([&] {
        if (!e || !blocks || !e->d_xchg) fail(SINKR_INVALID_ARGUMENT, "peer merge not set up");
        CK(cudaSetDevice(e->device));
        std::vector<uint8_t*> b(e->world);
        for (uint32_t q = 0; q < e->world; ++q) b[q] = static_cast<uint8_t*>(blocks[q]);
        peer_tables(e, b);
    });
}

void* sinkr_peer_block(sinkr_engine* e) { return e ? e->d_xchg : nullptr; }

sinkr_status sinkr_routed_decode_peer_async(sinkr_engine* e, const float* d_queries, size_t layer,
                                            const sinkr_routing_config* config,
                                            const sinkr_engine_options* options,
                                            float* d_outputs) {
    return guard([&] {
        if (!e || !d_queries || !d_outputs) fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (!e->d_peer_xchg) fail(SINKR_INVALID_ARGUMENT, "peer merge not set up (sinkr_peer_open)");
        if (e->peer_poisoned)
            fail(SINKR_LOGIC_ERROR, "peer merge disabled after a watchdog timeout (set it up again)");
        CK(cudaSetDevice(e->device));
        stage_params(e, layer, config, options, false);
        run_graph(e, d_queries, d_outputs, 3);
    });
}

sinkr_status sinkr_last_step_stats(sinkr_engine* e, uint32_t* kernel_launches, float* decode_ms,
                                   float* step_ms) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        CK(cudaStreamSynchronize(e->stream));
        if (kernel_launches) *kernel_launches = e->last_launches;
        if (decode_ms) {
            *decode_ms = 0.f;
            if (e->timing)
                CK(cudaEventElapsedTime(decode_ms, e->ev[e->fused ? 0 : 1], e->ev[e->fused ? 3 : 2]));
        }
        if (step_ms) {
            *step_ms = 0.f;
            if (e->timing || e->step_events)
                CK(cudaEventElapsedTime(step_ms, e->ev[0], e->ev[3]));
        }
    });
}

sinkr_status sinkr_step_io_buffers(sinkr_engine* e, float** queries, const float** outputs) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        if (queries) *queries = reinterpret_cast<float*>(e->h_in + e->off_q);
        if (outputs) *outputs = reinterpret_cast<const float*>(e->h_res);
    });
}

sinkr_status sinkr_step_io_bytes(sinkr_engine* e, size_t* h2d, size_t* d2h) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        if (h2d) *h2d = e->in_bytes;
        if (d2h) *d2h = e->res_bytes;
    });
}

// debug: cycle stamps of the last fused step (lead CTA), valid after fetch_step_info
extern "C" sinkr_status sinkr_debug_trace(sinkr_engine* e, unsigned long long* out) {
    return guard([&] {
        if (!e->d_trace) fail(SINKR_INVALID_ARGUMENT, "tracing disabled (SINKR_TRACE=1)");
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaMemcpy(out, e->d_trace, e->grid * 8 * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemset(e->d_trace, 0, e->grid * 8 * 8));
    });
}

// debug: touch the K and V regions of `layer` with one 4-byte load every
// `stride` bytes on the engine stream (cold-start experiments: warms address
// translation for the region without pulling it into L2 beyond a line/stride)
__global__ void debug_touch_kernel(const uint8_t* k, const uint8_t* v, size_t bytes, size_t stride,
                                   unsigned int* sink) {
    unsigned int acc = 0;
    for (size_t off = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * stride; off < bytes;
         off += (size_t)gridDim.x * blockDim.x * stride)
        acc += *reinterpret_cast<const volatile unsigned int*>(k + off) +
               *reinterpret_cast<const volatile unsigned int*>(v + off);
    if (acc == 0x9e3779b9u) *sink = acc;
}

extern "C" sinkr_status sinkr_debug_touch(sinkr_engine* e, size_t layer, size_t stride) {
    return guard([&] {
        const size_t bytes = e->U * e->cap * e->D * 2;
        const uint8_t* k = reinterpret_cast<const uint8_t*>(e->d_k) + layer * bytes;
        const uint8_t* v = reinterpret_cast<const uint8_t*>(e->d_v) + layer * bytes;
        debug_touch_kernel<<<148, 128, 0, e->stream>>>(k, v, bytes, stride,
                                                       reinterpret_cast<unsigned int*>(e->d_norm64));
        CK(cudaGetLastError());
    });
}

extern "C" sinkr_status sinkr_debug_stamps(sinkr_engine* e, unsigned long long* out, int n) {
    return guard([&] {
        const auto* st = reinterpret_cast<const unsigned long long*>(e->h_res + e->off_status + 48);
        for (int i = 0; i < n && i < 32; ++i) out[i] = st[i];
    });
}

sinkr_status sinkr_set_timing(sinkr_engine* e, int enabled) {
    return guard([&] {
        if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
        e->timing = enabled != 0;
    });
}

}  // extern "C"

// ---- pipelined multi-slot f32 append (snapshot replay) ----------------------
namespace sinkr {
namespace host {

void append_slots_f32(sinkr_engine* e, size_t seq, size_t rows, const SlotReader& read) {
    if (!e) fail(SINKR_INVALID_ARGUMENT, "null engine");
    CK(cudaSetDevice(e->device));
    const size_t H = e->cfg.num_kv_heads, nslots = e->layers * H, D = e->D, n = rows * D;
    if (rows == 0 || nslots == 0) return;
    for (size_t l = 0; l < e->layers; ++l)
        for (size_t h = 0; h < H; ++h) {
            check_slot(e, seq, l, h);
            if (e->len[e->slot_index(l, seq, h)] + rows > e->cap)
                fail(SINKR_RUNTIME_ERROR, "kv cache overflow: slot at capacity " + std::to_string(e->cap));
        }
    struct Res {
        cudaStream_t s = nullptr;
        float* hp[2] = {};
        float* dp = nullptr;
        double* d_n64 = nullptr;
        cudaEvent_t ev[2] = {};
        ~Res() {
            if (s) cudaStreamSynchronize(s);  // no copy may still read the pinned buffers
            for (auto* p : hp)
                if (p) cudaFreeHost(p);
            if (dp) cudaFree(dp);
            if (d_n64) cudaFree(d_n64);
            for (auto v : ev)
                if (v) cudaEventDestroy(v);
        }
    } r;
    r.s = e->stream;
    const size_t nv = (n + 3) / 4 * 4;  // 16-byte aligned halves
    for (auto*& p : r.hp) CK(cudaHostAlloc(reinterpret_cast<void**>(&p), 2 * nv * 4, cudaHostAllocDefault));
    CK(cudaMalloc(&r.dp, 4 * nv * 4));
    CK(cudaMalloc(&r.d_n64, nslots * 8));
    for (auto& v : r.ev) CK(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
    std::vector<uint8_t> first(nslots, 0);
    read(0, 0, r.hp[0], r.hp[0] + nv);
    for (size_t i = 0; i < nslots; ++i) {
        const int b = (int)(i & 1);
        const size_t l = i / H, h = i % H, idx = e->slot_index(l, seq, h);
        float* dk = r.dp + 2 * nv * b;
        float* dv = dk + nv;
        CK(cudaMemcpyAsync(dk, r.hp[b], 2 * nv * 4, cudaMemcpyHostToDevice, e->stream));
        const size_t off = (e->row_base(l, seq, h) + e->len[idx]) * D;
        const int grid = (int)std::min<size_t>((n / 4 + 255) / 256 + 1, (size_t)e->num_sms * 8);
        dev::f32_to_bf16_kernel<<<grid, 256, 0, e->stream>>>(dk, e->d_k + off, n);
        dev::f32_to_bf16_kernel<<<grid, 256, 0, e->stream>>>(dv, e->d_v + off, n);
        if (e->len[idx] == 0) {
            first[i] = 1;
            dev::anchor_capture_kernel<<<1, 32, 0, e->stream>>>(e->d_k + idx * e->cap * D, (uint32_t)D,
                                                                 e->d_anchor + idx * D, e->d_anchor_norm + idx,
                                                                 r.d_n64 + i);
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(r.ev[b], e->stream));
        if (i + 1 < nslots) {
            CK(cudaEventSynchronize(r.ev[b ^ 1]));  // slot i-1 done: its pinned buffer is free
            read((i + 1) / H, (i + 1) % H, r.hp[b ^ 1], r.hp[b ^ 1] + nv);
        }
    }
    std::vector<double> norms(nslots, 0.0);
    CK(cudaMemcpyAsync(norms.data(), r.d_n64, nslots * 8, cudaMemcpyDeviceToHost, e->stream));
    CK(cudaStreamSynchronize(e->stream));
    for (size_t i = 0; i < nslots; ++i) {
        const size_t idx = e->slot_index(i / H, seq, i % H);
        if (first[i]) {
            CK(cudaMemcpy(e->h_anchor.data() + idx * D, e->d_anchor + idx * D, D * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(e->h_anchor_norm.data() + idx, e->d_anchor_norm + idx, 4, cudaMemcpyDeviceToHost));
            if (norms[i] < 1e-12) fail(SINKR_RUNTIME_ERROR, "degenerate anchor: first-token key norm below 1e-12");
            e->anchored[idx] = 1;
        }
        e->len[idx] += rows;
        e->dlen_dirty = true;
    }
}

}  // namespace host
}  // namespace sinkr
