// NEXT #1: entropy coding of the integer latents (PAPER.md:1386-1387:
// "flattens our integer latent matrix for each attribute ... encoded using standard entropy
// coding approaches such as arithmetic coding").  The paper's coder is a single sequential
// arithmetic stream; to decode on the GPU we use the same kind of coder (an order-0
// static-model range/ANS coder) cut into independently decodable chunks and 32-way
// interleaved inside each chunk, so one warp decodes a chunk with one rANS state per lane.
//
// Stream format ("QAN2"), all little-endian:
//   u32 magic 'QAN2' | u32 n_sym | u32 n_chunks | u32 reserved
//   u16 freq[256]                    normalised to sum 4096 (PROB_BITS = 12); symbol = latent + 128
//   u32 word_off[n_chunks + 1]       chunk word offsets into words[]
//   u32 state[n_chunks][32]          initial decoder state of each lane
//   u16 lane_count[n_chunks][32]     renormalisation words of each lane
//   u16 words[]                      per chunk: lane 0's words in decoding order, lane 1's, ...
//                                    (padded to 4 bytes)
// Symbols are the category's latent matrix flattened row-major (k * n + i, k < L, i < n);
// chunk j holds symbols [j*CH, (j+1)*CH), CH = 8192; lane l of chunk j decodes symbols
// j*CH + 32 t + l for t = 0, 1, ... with its own rANS state (32-bit, in [2^16, 2^32)) and its
// own word sequence (16-bit renormalisation), so a lane never waits for the others.
#include <algorithm>
#include <cstring>
#include <vector>

#include "queen_internal.cuh"

namespace queen {

constexpr uint32_t ANS_MAGIC = 0x324e4151u;  // 'QAN2'
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
// One launch per frame (every category).  A block builds its category's slot table in shared
// memory straight from the stream's 256 frequencies: slot -> (f - 1) | latent byte << 12 |
// (slot - c) << 20, one 32-bit word.  Each warp then decodes one chunk, one rANS state per lane, from the
// chunk's words staged in shared memory; a lane's critical path per symbol is ONE shared load,
// one multiply-add, a compare and a select (no warp vote or shuffle).
//
// Bounds (every stream is wire input): the host passes each category's expected symbol and
// chunk counts (L * n, from the packet shape) and the stream's byte size.  A block whose
// header does not match (magic, n_sym, n_chunks, frequency sum) raises QUEEN_ERR_INDEX and
// writes nothing; a chunk whose word range lies outside the stream, or whose lane counts do
// not add up to it, raises it and writes nothing; every read stays inside the lane's range.
constexpr int ANS_WARPS = 8;
constexpr int ANS_STAGE = 4096;  // renormalisation words staged per warp (4 bits per symbol)
constexpr size_t ANS_SMEM = sizeof(uint16_t) * ANS_WARPS * (ANS_STAGE + 288);  // dynamic shared memory

struct AnsFrame {
    const unsigned char* stream[5];
    int L[5];
    int row0[5];          // first latent row of the category in the [sum L][n_pad] matrix
    int block0[6];        // first block of each category (prefix), block0[5] = total blocks
    uint32_t n_sym[5];    // host-expected symbols (L * n) and chunks of each category
    uint32_t n_chunks[5];
    uint32_t n_words[5];  // 16-bit renormalisation words the stream's byte size can hold
    int n, n_pad;
};

// Setup is two global round trips: (1) the header, the frequencies and the chunk's offsets,
// lane counts and states (all addressed by the host-expected counts, so in bounds whatever the
// header says); (2) the chunk's words, staged in shared memory while warp 0 scans the
// frequencies.  A slot's entry packs (f - 1) | byte << 12 | (slot - c) << 20, so a decode
// step is x' = (f - 1) * xs + (xs + (slot - c)): an AND and a LEA.HI side by side, then one IMAD.
__global__ void __launch_bounds__(ANS_WARPS * 32) k_ans_decode(const AnsFrame fr, int8_t* __restrict__ out,
                                                               DevFlags* fl) {
    __shared__ uint32_t s_tab[ANS_M];  // slot -> (f - 1) | latent byte << 12 | (slot - c) << 20
    __shared__ uint32_t s_c[257];
    extern __shared__ uint16_t s_words_dyn[];  // [ANS_WARPS][ANS_STAGE + 288]
    int cat = 0;
    while (cat < 4 && (int)blockIdx.x >= fr.block0[cat + 1]) ++cat;
    const unsigned char* stream = fr.stream[cat];
    const int n = fr.n, n_pad = fr.n_pad;
    const AnsHeader* h = reinterpret_cast<const AnsHeader*>(stream);
    const uint32_t n_sym = fr.n_sym[cat], n_chunks = fr.n_chunks[cat];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // round trip 1: header, frequencies (warp 0), this warp's chunk record
    const uint32_t chunk = (blockIdx.x - fr.block0[cat]) * ANS_WARPS + wid;
    const bool live = chunk < n_chunks;  // warp-uniform
    const uint32_t* woff = reinterpret_cast<const uint32_t*>(stream + sizeof(AnsHeader));
    const uint32_t* states = woff + n_chunks + 1;
    const uint16_t* lcount = reinterpret_cast<const uint16_t*>(states + (size_t)n_chunks * ANS_LANES);
    const uint16_t* words = lcount + (size_t)n_chunks * ANS_LANES;
    const bool hdr_ok = h->magic == ANS_MAGIC && h->n_sym == n_sym && h->n_chunks == n_chunks;
    uint32_t v[8];
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = h->freq[lane * 8 + q];
    }
    uint32_t c0 = 0, c1 = 0, cnt = 0, x = ANS_L;
    if (live) {
        c0 = woff[chunk];
        c1 = woff[chunk + 1];
        cnt = lcount[(size_t)chunk * ANS_LANES + lane];
        x = states[(size_t)chunk * ANS_LANES + lane];
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t nw = c1 - c0;
    const bool chunk_ok = live && hdr_ok && c0 <= c1 && c1 <= fr.n_words[cat] && nw == tot;  // warp-uniform
    if (live && hdr_ok && !chunk_ok && lane == 0) raise_flag(fl, FLAG_INDEX);
    const bool staged = chunk_ok && nw <= ANS_STAGE && n >= 32;
    uint16_t* sw = s_words_dyn + wid * (ANS_STAGE + 288);
    // round trip 2: the chunk's words into shared memory (coalesced, 8 loads in flight per lane)
    if (staged) {
        for (uint32_t q0 = 0; q0 < nw; q0 += 32 * 8) {
            uint16_t wv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                wv[u] = q < nw ? __ldg(words + c0 + q) : (uint16_t)0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t q = q0 + 32 * u + lane;
                if (q < nw) sw[q] = wv[u];
            }
        }
    }
    if (wid == 0) {  // exclusive scan of the 256 frequencies
        uint32_t sum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) sum += v[q];
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        uint32_t run = inc - sum;
#pragma unroll
        for (int q = 0; q < 8; ++q) { s_c[lane * 8 + q] = run; run += v[q]; }
        if (lane == 31) s_c[256] = run;
    }
    __syncthreads();
    if (!hdr_ok || s_c[256] != ANS_M) {  // bad header or corrupt frequency table (block-uniform)
        if (threadIdx.x == 0) raise_flag(fl, FLAG_INDEX);
        return;
    }
    {  // slot table: thread t fills slots [t*SPT, (t+1)*SPT): binary search once, then walk
        constexpr int SPT = ANS_M / (ANS_WARPS * 32);
        const uint32_t s0 = threadIdx.x * SPT;
        int lo = 0, hi = 256;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_c[mid] <= s0) lo = mid; else hi = mid;
        }
        uint32_t c_lo = s_c[lo], c_hi = s_c[lo + 1];
        for (uint32_t slot = s0; slot < s0 + SPT; ++slot) {
            while (slot >= c_hi) { ++lo; c_lo = c_hi; c_hi = s_c[lo + 1]; }
            s_tab[slot] = (c_hi - c_lo - 1u) | ((uint32_t)(uint8_t)(lo - 128) << 12) | ((slot - c_lo) << 20);
        }
    }
    __syncthreads();
    if (!chunk_ok) return;
    int8_t* cout = out + (size_t)fr.row0[cat] * n_pad;
    const uint32_t base = chunk * ANS_CHUNK;
    const uint32_t len = min((uint32_t)ANS_CHUNK, n_sym - base);
    const uint32_t k = (base + lane) / (uint32_t)n;
    uint32_t i = (base + lane) - k * (uint32_t)n;
    int8_t* op = cout + (size_t)k * n_pad + i;  // this lane's next output byte (row k, column i)
    const uint32_t mine = len > (uint32_t)lane ? (len - lane + 31) / 32 : 0u;  // this lane's symbols
    uint32_t ptr = incl - cnt, end = incl;  // this lane's words, relative to the chunk: [ptr, end)
    if (staged) {
        // common case: a renormalisation is a select on a word already in a register -- no
        // branch.  (The staging area has 288 words of slack: a lane's pointer advances at
        // most once per step, so even a corrupt stream never reads past it; the final check
        // flags it.)  The lane's column wraps into the next row once every ~n/32 steps, at step
        // tw: steps run in segments that end there, so the hot loop has no row-wrap test.
        const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(sw);
        uint32_t wa = wbase + 2u * ptr;             // shared address of the lane's next word
        uint32_t tw = ((uint32_t)n - i + 31) / 32;  // step after which the column passes n
        uint32_t t_i = 0;                           // step at which the lane was at column i
        // the lane's next word waits in a register and is reloaded only after a renormalisation
        // consumed it (predicated, a step ahead of its use): one shared load per renormalisation,
        // not one per step.  (Lanes of high-entropy chunks advance in lockstep through regions
        // spaced by multiples of 32 banks, so per-step word loads were 10-way bank conflicts.)
        uint16_t wn;
        asm("ld.shared.u16 %0, [%1];" : "=h"(wn) : "r"(wa));
        auto step = [&](int u) {
            const uint32_t e = s_tab[x & (ANS_M - 1)];
            const uint32_t xs = x >> ANS_PROB_BITS;
            const uint32_t xd = (e & 0xfffu) * xs + (xs + (e >> 20));  // f * xs + slot - c
            const bool need = xd < ANS_L;
            x = need ? ((xd << 16) | (uint32_t)wn) : xd;
            wa += need ? 2u : 0u;
            if (need) asm("ld.shared.u16 %0, [%1];" : "=h"(wn) : "r"(wa));
            op[32 * u] = (int8_t)(e >> 12);
        };
        for (uint32_t t = 0; t < mine;) {
            const uint32_t tend = min(mine, tw);
            for (; t + 4 <= tend; t += 4) {
                step(0);
                step(1);
                step(2);
                step(3);
                op += 128;
            }
            for (; t < tend; ++t) {
                step(0);
                op += 32;
            }
            if (t == tw) {  // column i + 32 (tw - t_i) >= n: continue in the next row
                i = i + 32 * (tw - t_i) - (uint32_t)n;
                op += n_pad - n;
                t_i = tw;
                tw += ((uint32_t)n - i + 31) / 32;
            }
        }
        ptr = (wa - wbase) >> 1;
    } else {
        // more words than the staging area (> 4 bits per symbol), or rows shorter than a warp:
        // read the words from the stream
        ptr += c0;
        end += c0;
        for (uint32_t t = 0; t < mine; ++t) {
            const uint32_t e = s_tab[x & (ANS_M - 1)];
            const uint32_t xs = x >> ANS_PROB_BITS;
            x = (e & 0xfffu) * xs + (xs + (e >> 20));
            *op = (int8_t)(e >> 12);
            if (x < ANS_L) {
                x = (x << 16) | (ptr < end ? (uint32_t)__ldg(words + ptr) : 0u);
                ++ptr;
            }
            i += 32;
            op += 32;
            while (i >= (uint32_t)n) { i -= (uint32_t)n; op += n_pad - n; }
        }
    }
    if (ptr != end || x != ANS_L) raise_flag(fl, FLAG_INDEX);  // corrupt / mismatched stream
}

cudaError_t init_entropy_attributes() {
    return cudaFuncSetAttribute(k_ans_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ANS_SMEM);
}

// host: expected counts of one category's stream (L * n symbols), and the renormalisation
// words its byte size can hold; false if the stream cannot even hold its header and tables
static bool ans_expect(int L, int n, int64_t bytes, uint32_t& n_sym, uint32_t& n_chunks, uint32_t& n_words) {
    const uint64_t ns = (uint64_t)L * (uint64_t)n;
    if (ns > 0xffffffffull) return false;
    n_sym = (uint32_t)ns;
    n_chunks = (uint32_t)((ns + ANS_CHUNK - 1) / ANS_CHUNK);
    const int64_t fixed = (int64_t)sizeof(AnsHeader) + 4 * ((int64_t)n_chunks + 1) + 6 * (int64_t)ANS_LANES * n_chunks;
    if (bytes < fixed) return false;
    const int64_t nw = (bytes - fixed) / 2;
    n_words = (uint32_t)std::min<int64_t>(nw, 0xffffffffll);
    return true;
}

// returns cudaErrorInvalidValue when a stream is too small for its (L, n) (host-detectable)
cudaError_t launch_ans_decode_frame(const void* const streams[5], const int64_t bytes[5], const int L[5], int n,
                                    int n_pad, int8_t* out, DevFlags* fl, cudaStream_t s) {
    AnsFrame fr{};
    fr.n = n;
    fr.n_pad = n_pad;
    int row = 0, blk = 0;
    for (int c = 0; c < 5; ++c) {
        fr.stream[c] = static_cast<const unsigned char*>(streams[c]);
        fr.L[c] = (streams[c] && L[c] > 0) ? L[c] : 0;
        fr.row0[c] = row;
        fr.block0[c] = blk;
        row += L[c] > 0 ? L[c] : 0;
        if (fr.L[c] == 0 || n == 0) continue;
        if (!ans_expect(fr.L[c], n, bytes[c], fr.n_sym[c], fr.n_chunks[c], fr.n_words[c])) return cudaErrorInvalidValue;
        blk += (int)((fr.n_chunks[c] + ANS_WARPS - 1) / ANS_WARPS);
    }
    fr.block0[5] = blk;
    if (blk == 0) return cudaSuccess;
    k_ans_decode<<<blk, ANS_WARPS * 32, ANS_SMEM, s>>>(fr, out, fl);
    return cudaGetLastError();
}

cudaError_t launch_ans_decode(const void* stream_dev, int64_t bytes, int L, int n, int n_pad, int8_t* out,
                              DevFlags* fl, cudaStream_t s) {
    const void* streams[5] = {stream_dev, nullptr, nullptr, nullptr, nullptr};
    const int64_t b5[5] = {bytes, 0, 0, 0, 0};
    const int Ls[5] = {L, 0, 0, 0, 0};
    return launch_ans_decode_frame(streams, b5, Ls, n, n_pad, out, fl, s);
}

// ---------------------------------------------------------------- host encoder
// Produces exactly the stream the decoder consumes: per chunk and lane, the lane's symbols
// are encoded in the reverse of decoding order (t descending); the words its pre-encode
// renormalisations emit are reversed at the end so the decoder reads them forward.
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
    std::vector<uint16_t> lcount((size_t)n_chunks * ANS_LANES, 0);
    std::vector<uint16_t> words;
    std::vector<uint16_t> rev;
    for (uint32_t c = 0; c < n_chunks; ++c) {
        const uint64_t base = (uint64_t)c * ANS_CHUNK;
        const uint32_t len = (uint32_t)std::min<uint64_t>(ANS_CHUNK, n_sym - base);
        woff[c] = (uint32_t)words.size();
        for (int l = 0; l < ANS_LANES; ++l) {
            uint32_t x = ANS_L;
            rev.clear();
            const uint32_t mine = len > (uint32_t)l ? (len - l + 31) / 32 : 0u;
            for (int64_t t = (int64_t)mine - 1; t >= 0; --t) {
                const uint64_t flat = base + (uint64_t)t * 32 + l;
                const int k = (int)(flat / (uint64_t)n), i = (int)(flat % (uint64_t)n);
                const uint32_t s = (uint8_t)((int)lat[(size_t)k * n_pad + i] + 128);
                const uint32_t f = h.freq[s];
                const uint64_t xmax = (uint64_t)((ANS_L >> ANS_PROB_BITS) << 16) * f;  // f = 4096 -> 2^32
                if ((uint64_t)x >= xmax) {
                    rev.push_back((uint16_t)(x & 0xffffu));
                    x >>= 16;
                }
                x = ((x / f) << ANS_PROB_BITS) + (x % f) + cum[s];
            }
            states[(size_t)c * ANS_LANES + l] = x;
            lcount[(size_t)c * ANS_LANES + l] = (uint16_t)rev.size();
            for (size_t q = rev.size(); q-- > 0;) words.push_back(rev[q]);
        }
    }
    woff[n_chunks] = (uint32_t)words.size();
    const size_t bytes = sizeof(AnsHeader) + 4 * woff.size() + 4 * states.size() + 2 * lcount.size() +
                         ((2 * words.size() + 3) & ~size_t(3));
    out.assign(bytes, 0);
    unsigned char* o = out.data();
    std::memcpy(o, &h, sizeof(h));
    o += sizeof(h);
    std::memcpy(o, woff.data(), 4 * woff.size());
    o += 4 * woff.size();
    std::memcpy(o, states.data(), 4 * states.size());
    o += 4 * states.size();
    std::memcpy(o, lcount.data(), 2 * lcount.size());
    o += 2 * lcount.size();
    if (!words.empty()) std::memcpy(o, words.data(), 2 * words.size());
    return bytes;
}

}  // namespace queen
