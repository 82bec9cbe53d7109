// map.cpp -- map blob parsing and packing of the factorised network for eval_map.
//
// Network shape: classifier 4 -> 32 -> 32 -> 1, regressor
// 4 -> 32 -> 32 -> 32 -> 32 -> 32 -> 6, tanh hidden layers, linear outputs.
// The bf16 weights are re-laid-out into the tcgen05 canonical K-major, no-swizzle
// shared-memory layout: element (n, k) of a B operand with K columns lives at
//   (n/8) * (K/8)*128 + (k/8) * 128 + (n%8) * 16 + (k%8) * 2   bytes,
// i.e. 8-row x 16-byte core matrices, adjacent along K (LBO = 128 B) and stacked
// along N (SBO = K/8 * 128 B).  The input layer's operand repeats W along K so one
// K=16 MMA consumes the exact bf16 hi/mid/lo split of the 4 inputs: k 0..3, 4..7, 8..11 = W.
#include <algorithm>
#include <cmath>
#include <cstring>

#include <cuda_runtime.h>

#include "host.h"

plt_map::~plt_map() {
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    for (auto& kv : dev_image) {
        if (!kv.second) continue;
        cudaSetDevice(kv.first);
        cudaFree(kv.second);
    }
    cudaSetDevice(cur);
}

namespace plt {

namespace {
[[noreturn]] void fail(plt_status c, const std::string& m) { throw Error{c, m}; }

struct Reader {
    const uint8_t* p; size_t n, off = 0;
    void need(size_t k, const char* what) {
        if (off + k > n) fail(PLT_E_PARSE, std::string("map blob truncated while reading ") + what);
    }
    template <typename T> T get(const char* what) {
        need(sizeof(T), what);
        T v;
        std::memcpy(&v, p + off, sizeof(T));
        off += sizeof(T);
        return v;
    }
};

uint16_t bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf16_to_f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Pack W (fo x fi, bf16 bits) and bias b (fo, fp32) into an N = n_pad, K = k_total operand.
// Input layer (k_total = 16): k 0..fi-1, fi..2fi-1, 2fi..3fi-1 = W (against the hi/mid/lo
// thirds of A), 3fi..3fi+2 = bias hi/mid/lo.  Hidden/output (k_total = 48): k 0..31 = W,
// 32..34 = bias hi/mid/lo, rest 0.  The 3-term bias split is exact for an fp32 bias.
void pack_operand(uint8_t* dst, const uint16_t* W, const float* b, int fo, int fi, int n_pad, int k_total,
                  bool input) {
    const int sbo = (k_total / 8) * 128;
    const int kb = input ? 3 * fi : 32;
    for (int nn = 0; nn < n_pad; ++nn)
        for (int k = 0; k < k_total; ++k) {
            uint16_t v = 0;
            if (nn < fo) {
                const float bh = bf16_to_f(bf16_rne(b[nn]));
                const float bm = bf16_to_f(bf16_rne(b[nn] - bh));
                if (k < kb) { if (input || k < fi) v = W[nn * fi + (k % fi)]; }
                else if (k == kb) v = bf16_rne(b[nn]);
                else if (k == kb + 1) v = bf16_rne(b[nn] - bh);
                else if (k == kb + 2) v = bf16_rne(b[nn] - bh - bm);
            }
            const size_t off = (size_t)(nn / 8) * sbo + (k / 8) * 128 + (nn % 8) * 16 + (k % 8) * 2;
            std::memcpy(dst + off, &v, 2);
        }
}
}  // namespace

plt_map* parse_map(const plt_lens* lens, const uint8_t* blob, size_t len) {
    Reader r{blob, len};
    r.need(8, "magic");
    if (std::memcmp(blob, "PLTMAP01", 8) != 0) fail(PLT_E_PARSE, "bad map magic (expected PLTMAP01)");
    r.off = 8;
    auto m = std::make_unique<plt_map>();
    const uint32_t ver = r.get<uint32_t>("version");
    if (ver != 1 && ver != 2) fail(PLT_E_PARSE, "unsupported map version " + std::to_string(ver));
    m->direction = r.get<uint32_t>("direction");
    m->path_id = r.get<uint64_t>("path_id");
    const uint32_t ncl = r.get<uint32_t>("n_cls_layers"), nrl = r.get<uint32_t>("n_reg_layers");
    if (ver >= 2) {   // version 2 records the input plane the map was trained on (rays' plane_z)
        m->plane_z = r.get<double>("plane_z_mm");
        if (!std::isfinite(m->plane_z)) fail(PLT_E_VALIDATION, "map input plane z must be finite");
        m->has_plane = true;
    }
    if (ncl != 3 || nrl != 6)
        fail(PLT_E_VALIDATION, "map must have 3 classifier and 6 regressor layers (P:391-392)");
    if (m->direction > 1) fail(PLT_E_VALIDATION, "map direction must be 0 or 1");
    float norm[20];
    for (int i = 0; i < 20; ++i) norm[i] = r.get<float>("normalisation");
    for (int d = 0; d < 4; ++d) {
        if (!(norm[4 + d] > norm[d])) fail(PLT_E_VALIDATION, "input normalisation needs hi > lo");
        m->params.in_lo[d] = norm[d];
        m->params.in_scale[d] = (float)(2.0 / ((double)norm[4 + d] - (double)norm[d]));
    }
    for (int d = 0; d < 6; ++d) { m->params.out_mid[d] = norm[8 + d]; m->params.out_half[d] = norm[14 + d]; }

    static const int cls_dims[4] = {4, 32, 32, 1};
    static const int reg_dims[7] = {4, 32, 32, 32, 32, 32, 6};
    MapLayout& L = m->layout;
    uint32_t off = 0;
    auto place = [&](int n_pad, int k_total) { uint32_t o = off; off += (uint32_t)(n_pad * k_total * 2); return o; };
    L.cls_w[0] = place(32, 16); L.cls_w[1] = place(32, 48);
    L.reg_w[0] = place(32, 16);
    for (int l = 1; l < 5; ++l) L.reg_w[l] = place(32, 48);
    L.reg_out = place(16, 48);
    L.out_off = (off + 15u) & ~15u;
    L.total_bytes = (L.out_off + 4u * kOutFloats + 15u) & ~15u;
    m->image.assign(L.total_bytes, 0);
    float* outw = reinterpret_cast<float*>(m->image.data() + L.out_off);

    // read both heads: per layer W (bf16, [fo][fi]) and b (fp32, [fo])
    std::vector<uint16_t> Wl[2][6];
    std::vector<float> bl[2][6];
    for (int head = 0; head < 2; ++head) {
        const int nl = head == 0 ? 3 : 6;
        const int* dims = head == 0 ? cls_dims : reg_dims;
        for (int l = 0; l < nl; ++l) {
            const uint32_t fo = r.get<uint32_t>("layer out"), fi = r.get<uint32_t>("layer in");
            if ((int)fo != dims[l + 1] || (int)fi != dims[l])
                fail(PLT_E_VALIDATION, std::string(head ? "regressor" : "classifier") + " layer " + std::to_string(l) +
                                           " has dims " + std::to_string(fi) + "->" + std::to_string(fo) +
                                           ", expected " + std::to_string(dims[l]) + "->" + std::to_string(dims[l + 1]));
            std::vector<uint16_t>& W = Wl[head][l];
            W.resize(fo * fi);
            r.need(2 * W.size(), "weights");
            std::memcpy(W.data(), blob + r.off, 2 * W.size());
            r.off += 2 * W.size();
            std::vector<float>& b = bl[head][l];
            b.resize(fo);
            for (uint32_t o = 0; o < fo; ++o) b[o] = r.get<float>("bias");
        }
    }
    // Classifier first hidden layer: order its 32 units by their influence on the logit,
    // s_j = sum_i |w3_i| |W2_ij| (a bound on d logit / d h1_j), most influential first.
    // The kernel evaluates the first 16 with the accurate tanh and the rest with MUFU
    // tanh.approx.  Permuting hidden units (W1 rows, b1,
    // W2 columns) leaves the network's function unchanged.
    {
        const std::vector<uint16_t>&W2 = Wl[0][1], &w3 = Wl[0][2];
        double sens[32];
        for (int j = 0; j < 32; ++j) {
            sens[j] = 0.0;
            for (int i = 0; i < 32; ++i) sens[j] += std::fabs((double)bf16_to_f(w3[i])) * std::fabs((double)bf16_to_f(W2[i * 32 + j]));
        }
        int perm[32];
        for (int j = 0; j < 32; ++j) perm[j] = j;
        std::stable_sort(perm, perm + 32, [&](int a, int b) { return sens[a] > sens[b]; });
        std::vector<uint16_t> W1 = Wl[0][0], W2p = W2;
        std::vector<float> b1 = bl[0][0];
        for (int nw = 0; nw < 32; ++nw) {
            const int od = perm[nw];
            for (int k = 0; k < 4; ++k) W1[nw * 4 + k] = Wl[0][0][od * 4 + k];
            b1[nw] = bl[0][0][od];
            for (int i = 0; i < 32; ++i) W2p[i * 32 + nw] = W2[i * 32 + od];
        }
        Wl[0][0] = W1; bl[0][0] = b1; Wl[0][1] = W2p;
    }
    for (int head = 0; head < 2; ++head) {
        const int nl = head == 0 ? 3 : 6;
        const int* dims = head == 0 ? cls_dims : reg_dims;
        for (int l = 0; l < nl; ++l) {
            const uint32_t fo = (uint32_t)dims[l + 1], fi = (uint32_t)dims[l];
            const std::vector<uint16_t>& W = Wl[head][l];
            const std::vector<float>& b = bl[head][l];
            if (head == 1 && l + 1 == nl) {   // regressor output layer: N = 6 padded to 16, K = 48
                pack_operand(m->image.data() + L.reg_out, W.data(), b.data(), (int)fo, (int)fi, 16, 48, false);
                continue;
            }
            if (l + 1 == nl) {   // classifier output layer: fp32 block
                for (uint32_t k = 0; k < fi; ++k) outw[kOutClsW + k] = m->params.cls_w3[k] = bf16_to_f(W[k]);
                outw[kOutClsB] = m->params.cls_b3 = b[0];
                continue;
            }
            const uint32_t woff = head == 0 ? L.cls_w[l] : L.reg_w[l];
            pack_operand(m->image.data() + woff, W.data(), b.data(), (int)fo, (int)fi, 32, l == 0 ? 16 : 48, l == 0);
        }
    }
    if (lens) {
        try {
            compile_path(*lens, m->path_id, (int)m->direction);
        } catch (const Error& e) {
            fail(PLT_E_VALIDATION, "map path id does not fit the lens: " + e.msg);
        }
    }
    return m.release();
}

}  // namespace plt
