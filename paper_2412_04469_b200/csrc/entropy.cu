// NEXT #1: entropy coding of the integer latents (PAPER.md:1386-1387:
// "flattens our integer latent matrix for each attribute ... encoded using standard entropy
// coding approaches such as arithmetic coding").  The paper's coder is a single sequential
// arithmetic stream; to decode on the GPU we use the same kind of coder (an order-0
// static-model range/ANS coder) cut into independently decodable chunks and 32-way
// interleaved inside each chunk, so one warp decodes a chunk with one rANS state per lane.
//
// Stream format ("QANS"), all little-endian:
//   u32 magic 'QANS' | u32 n_sym | u32 n_chunks | u32 reserved
//   u16 freq[256]                    normalised to sum 4096 (PROB_BITS = 12); symbol = latent + 128
//   u32 word_off[n_chunks + 1]       chunk word offsets into words[]
//   u32 state[n_chunks][32]          initial decoder state of each lane
//   u16 words[]                      renormalisation words in decoding order (padded to 4 bytes)
// Symbols are the category's latent matrix flattened row-major (k * n + i, k < L, i < n);
// chunk j holds symbols [j*CH, (j+1)*CH), CH = 8192; lane l of chunk j decodes symbols
// j*CH + 32 t + l for t = 0, 1, ...  rANS: 32-bit state in [2^16, 2^32), 16-bit renormalisation.
#include <cstring>
#include <vector>

#include "queen_internal.cuh"

namespace queen {

constexpr uint32_t ANS_MAGIC = 0x534e4151u;  // 'QANS'
constexpr int ANS_PROB_BITS = 12;
constexpr uint32_t ANS_M = 1u << ANS_PROB_BITS;
constexpr uint32_t ANS_L = 1u << 16;
constexpr int ANS_LANES = 32;
constexpr int ANS_CHUNK = 32 * 256;  // 8192 symbols: chunk count vs per-chunk state overhead

struct AnsHeader {
    uint32_t magic, n_sym, n_chunks, reserved;
    uint16_t freq[256];
};
static_assert(sizeof(AnsHeader) == 528, "AnsHeader layout");

// deterministic normalisation of the symbol counts to a table summing to ANS_M
static void normalise(const uint64_t cnt[256], uint64_t total, uint16_t f[256]) {
    int64_t sum = 0;
    int best = -1;
    for (int s = 0; s < 256; ++s) {
        f[s] = 0;
        if (!cnt[s]) continue;
        uint64_t v = cnt[s] * ANS_M / total;
        if (v == 0) v = 1;
        f[s] = (uint16_t)v;
        sum += (int64_t)v;
        if (best < 0 || cnt[s] > cnt[best]) best = s;
    }
    if (best < 0) return;
    if (sum <= (int64_t)ANS_M) {
        f[best] = (uint16_t)((int64_t)f[best] + ((int64_t)ANS_M - sum));
        return;
    }
    while (sum > (int64_t)ANS_M) {  // too many rare symbols bumped to 1: take from the largest
        int m = -1;
        for (int s = 0; s < 256; ++s)
            if (f[s] > 1 && (m < 0 || f[s] > f[m])) m = s;
        --f[m];
        --sum;
    }
}

// ---------------------------------------------------------------- device decoder
// Two launches per frame: k_ans_table builds every category's slot tables once (slot ->
// f | (slot - c) << 16 as u32, and slot -> the decoded int8 latent, 20 KB per category, in the
// workspace); k_ans_decode copies its category's tables to shared memory and decodes, one warp
// per chunk, one rANS state per lane: a decode step is ONE shared load + a multiply-add on the
// state's critical path (the symbol byte is looked up beside it).
constexpr int ANS_WARPS = 4;

struct AnsFrame {
    const unsigned char* stream[5];
    int L[5];
    int row0[5];          // first latent row of the category in the [sum L][n_pad] matrix
    int block0[6];        // first block of each category (prefix), block0[5] = total blocks
    int n, n_pad;
    const uint32_t* table;  // [5][ANS_M] (f | (slot - c) << 16), then [5][ANS_M] int8 symbols (k_ans_table)
};

__global__ void __launch_bounds__(256) k_ans_table(const AnsFrame fr, uint32_t* __restrict__ table, DevFlags* fl) {
    __shared__ uint16_t s_f[256];
    __shared__ uint32_t s_c[257];
    const int cat = blockIdx.y;
    if (fr.L[cat] == 0) return;
    const AnsHeader* h = reinterpret_cast<const AnsHeader*>(fr.stream[cat]);
    for (int q = threadIdx.x; q < 256; q += blockDim.x) s_f[q] = h->freq[q];
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 frequencies by one warp
        uint32_t v[8], sum = 0;
        for (int q = 0; q < 8; ++q) { v[q] = s_f[threadIdx.x * 8 + q]; sum += v[q]; }
        uint32_t inc = sum;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (threadIdx.x >= o) inc += y;
        }
        uint32_t run = inc - sum;
        for (int q = 0; q < 8; ++q) { s_c[threadIdx.x * 8 + q] = run; run += v[q]; }
        if (threadIdx.x == 31) s_c[256] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0 && s_c[256] != ANS_M) raise_flag(fl, FLAG_INDEX);  // corrupt table
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;  // symbol s with c[s] <= slot < c[s+1]
    if (slot >= ANS_M) return;
    int lo = 0, hi = 256;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (s_c[mid] <= slot) lo = mid; else hi = mid;
    }
    const uint32_t f = s_f[lo];
    table[(size_t)cat * ANS_M + slot] = f | ((slot - s_c[lo]) << 16);
    reinterpret_cast<int8_t*>(table + 5 * ANS_M)[(size_t)cat * ANS_M + slot] = (int8_t)(lo - 128);
}

__global__ void __launch_bounds__(ANS_WARPS * 32) k_ans_decode(const AnsFrame fr, int8_t* __restrict__ out, DevFlags* fl) {
    __shared__ uint32_t s_tab[ANS_M];
    __shared__ int8_t s_sym[ANS_M];
    int cat = 0;
    while (cat < 4 && (int)blockIdx.x >= fr.block0[cat + 1]) ++cat;
    const unsigned char* stream = fr.stream[cat];
    const int L = fr.L[cat], n = fr.n, n_pad = fr.n_pad;
    const AnsHeader* h = reinterpret_cast<const AnsHeader*>(stream);
    const uint32_t n_sym = h->n_sym, n_chunks = h->n_chunks;
    if (threadIdx.x == 0 && (h->magic != ANS_MAGIC || n_sym != (uint32_t)L * (uint32_t)n)) raise_flag(fl, FLAG_INDEX);
    {
        const uint4* src = reinterpret_cast<const uint4*>(fr.table + (size_t)cat * ANS_M);
        uint4* dst = reinterpret_cast<uint4*>(s_tab);
        for (int q = threadIdx.x; q < ANS_M / 4; q += blockDim.x) dst[q] = __ldg(src + q);
        const uint4* ssrc = reinterpret_cast<const uint4*>(reinterpret_cast<const int8_t*>(fr.table + 5 * ANS_M) +
                                                           (size_t)cat * ANS_M);
        for (int q = threadIdx.x; q < ANS_M / 16; q += blockDim.x) reinterpret_cast<uint4*>(s_sym)[q] = __ldg(ssrc + q);
    }
    __syncthreads();
    const uint32_t chunk = (blockIdx.x - fr.block0[cat]) * ANS_WARPS + (threadIdx.x >> 5);
    if (chunk >= n_chunks) return;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t* woff = reinterpret_cast<const uint32_t*>(stream + sizeof(AnsHeader));
    const uint32_t* states = woff + n_chunks + 1;
    const uint16_t* words = reinterpret_cast<const uint16_t*>(states + (size_t)n_chunks * ANS_LANES);
    int8_t* cout = out + (size_t)fr.row0[cat] * n_pad;
    uint32_t x = states[(size_t)chunk * ANS_LANES + lane];
    uint32_t ptr = woff[chunk];
    const uint32_t end = woff[chunk + 1];
    const uint32_t base = chunk * ANS_CHUNK;
    const uint32_t len = min((uint32_t)ANS_CHUNK, n_sym - base);
    const uint32_t steps = (len + 31) / 32;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t k = (base + lane) / (uint32_t)n;
    uint32_t i = (base + lane) - k * (uint32_t)n;
    int8_t* op = cout + (size_t)k * n_pad + i;  // this lane's next output byte (row k, column i)
    // The chunk's renormalisation words are consumed in order, ~1 per step for the warp.
    // Keep a 128-word window in registers (4 words per lane: current 64 + next 64), so a
    // renormalisation is a shuffle, and the next 64 words load one window ahead.
    auto ld = [&](uint32_t w) -> uint32_t { return w < end ? (uint32_t)__ldg(words + w) : 0u; };
    uint32_t wbase = ptr;
    uint32_t c0 = ld(wbase + lane), c1 = ld(wbase + 32 + lane), n0 = ld(wbase + 64 + lane), n1 = ld(wbase + 96 + lane);
    for (uint32_t t = 0; t < steps; ++t) {
        const bool active = t * 32 + lane < len;
        const uint32_t slot = x & (ANS_M - 1);
        const uint32_t e = s_tab[slot];
        const uint32_t xn = (e & 0xffffu) * (x >> ANS_PROB_BITS) + (e >> 16);
        if (active) {
            x = xn;
            *op = s_sym[slot];
        }
        const bool need = active && x < ANS_L;
        const uint32_t m = __ballot_sync(0xffffffffu, need);
        if (m) {
            const uint32_t q = ptr - wbase + __popc(m & lt);  // window position of this lane's word (< 96)
            const uint32_t src = q & 31u;
            const uint32_t a0 = __shfl_sync(0xffffffffu, c0, src), a1 = __shfl_sync(0xffffffffu, c1, src);
            const uint32_t a2 = __shfl_sync(0xffffffffu, n0, src);
            const uint32_t wv = q < 32 ? a0 : (q < 64 ? a1 : a2);
            if (need) x = (x << 16) | wv;
            ptr += __popc(m);
            if (ptr - wbase >= 64) {  // slide the window by 64 words
                wbase += 64;
                c0 = n0;
                c1 = n1;
                n0 = ld(wbase + 64 + lane);
                n1 = ld(wbase + 96 + lane);
            }
        }
        i += 32;  // next symbol of this lane: flat index + 32
        op += 32;
        while (i >= (uint32_t)n) { i -= (uint32_t)n; op += n_pad - n; }
    }
    if (ptr != end || x != ANS_L) raise_flag(fl, FLAG_INDEX);  // corrupt / mismatched stream
}

cudaError_t launch_ans_decode_frame(const void* const streams[5], const int L[5], int n, int n_pad, int8_t* out,
                                    uint32_t* table, DevFlags* fl, cudaStream_t s) {
    AnsFrame fr{};
    fr.n = n;
    fr.n_pad = n_pad;
    fr.table = table;
    int row = 0, blk = 0;
    for (int c = 0; c < 5; ++c) {
        fr.stream[c] = static_cast<const unsigned char*>(streams[c]);
        fr.L[c] = (streams[c] && L[c] > 0) ? L[c] : 0;
        fr.row0[c] = row;
        fr.block0[c] = blk;
        row += L[c] > 0 ? L[c] : 0;
        const int64_t chunks = ((int64_t)fr.L[c] * n + ANS_CHUNK - 1) / ANS_CHUNK;
        blk += (int)((chunks + ANS_WARPS - 1) / ANS_WARPS);
    }
    fr.block0[5] = blk;
    if (blk == 0) return cudaSuccess;
    k_ans_table<<<dim3(ANS_M / 256, 5), 256, 0, s>>>(fr, table, fl);
    k_ans_decode<<<blk, ANS_WARPS * 32, 0, s>>>(fr, out, fl);
    return cudaGetLastError();
}

cudaError_t launch_ans_decode(const void* stream_dev, int L, int n, int n_pad, int8_t* out, uint32_t* table,
                              DevFlags* fl, cudaStream_t s) {
    const void* streams[5] = {stream_dev, nullptr, nullptr, nullptr, nullptr};
    const int Ls[5] = {L, 0, 0, 0, 0};
    return launch_ans_decode_frame(streams, Ls, n, n_pad, out, table, fl, s);
}

// ---------------------------------------------------------------- host encoder
// Produces exactly the stream the decoder consumes: per chunk, the symbols are encoded in
// the reverse of decoding order (t descending, lane descending); the words emitted by the
// pre-encode renormalisations are reversed at the end so the decoder reads them forward.
size_t ans_encode(const int8_t* lat, int L, int n, int n_pad, std::vector<unsigned char>& out) {
    const uint64_t n_sym = (uint64_t)L * (uint64_t)n;
    const uint32_t n_chunks = (uint32_t)((n_sym + ANS_CHUNK - 1) / ANS_CHUNK);
    AnsHeader h{};
    h.magic = ANS_MAGIC;
    h.n_sym = (uint32_t)n_sym;
    h.n_chunks = n_chunks;
    uint64_t cnt[256] = {0};
    for (int k = 0; k < L; ++k)
        for (int i = 0; i < n; ++i) ++cnt[(uint8_t)((int)lat[(size_t)k * n_pad + i] + 128)];
    normalise(cnt, n_sym ? n_sym : 1, h.freq);
    uint32_t cum[257];
    cum[0] = 0;
    for (int s = 0; s < 256; ++s) cum[s + 1] = cum[s] + h.freq[s];
    std::vector<uint32_t> woff(n_chunks + 1, 0), states((size_t)n_chunks * ANS_LANES, ANS_L);
    std::vector<uint16_t> words;
    std::vector<uint16_t> rev;
    for (uint32_t c = 0; c < n_chunks; ++c) {
        const uint64_t base = (uint64_t)c * ANS_CHUNK;
        const uint32_t len = (uint32_t)std::min<uint64_t>(ANS_CHUNK, n_sym - base);
        const uint32_t steps = (len + 31) / 32;
        uint32_t x[ANS_LANES];
        for (int l = 0; l < ANS_LANES; ++l) x[l] = ANS_L;
        rev.clear();
        for (int64_t t = (int64_t)steps - 1; t >= 0; --t)
            for (int l = ANS_LANES - 1; l >= 0; --l) {
                const uint64_t p = (uint64_t)t * 32 + l;
                if (p >= len) continue;
                const uint64_t flat = base + p;
                const int k = (int)(flat / (uint64_t)n), i = (int)(flat % (uint64_t)n);
                const uint32_t s = (uint8_t)((int)lat[(size_t)k * n_pad + i] + 128);
                const uint32_t f = h.freq[s];
                const uint64_t xmax = (uint64_t)((ANS_L >> ANS_PROB_BITS) << 16) * f;  // f = 4096 -> 2^32
                if ((uint64_t)x[l] >= xmax) {
                    rev.push_back((uint16_t)(x[l] & 0xffffu));
                    x[l] >>= 16;
                }
                x[l] = ((x[l] / f) << ANS_PROB_BITS) + (x[l] % f) + cum[s];
            }
        woff[c] = (uint32_t)words.size();
        for (size_t q = rev.size(); q-- > 0;) words.push_back(rev[q]);
        for (int l = 0; l < ANS_LANES; ++l) states[(size_t)c * ANS_LANES + l] = x[l];
    }
    woff[n_chunks] = (uint32_t)words.size();
    const size_t bytes = sizeof(AnsHeader) + 4 * woff.size() + 4 * states.size() + ((2 * words.size() + 3) & ~size_t(3));
    out.assign(bytes, 0);
    unsigned char* o = out.data();
    std::memcpy(o, &h, sizeof(h));
    o += sizeof(h);
    std::memcpy(o, woff.data(), 4 * woff.size());
    o += 4 * woff.size();
    std::memcpy(o, states.data(), 4 * states.size());
    o += 4 * states.size();
    if (!words.empty()) std::memcpy(o, words.data(), 2 * words.size());
    return bytes;
}

}  // namespace queen
