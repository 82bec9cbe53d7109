// lens.cpp -- host lens layer: prescription parsing/validation, glass models, ABCD
// paraxial matrices, path-program compilation and two-bounce ghost enumeration.
//
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; readings A1..A30 of
// SURVEY.md §8(c) are restated in DESIGN.md.
#include <array>
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "host.h"

namespace plt {

namespace {
constexpr double kLambdaF = 0.4861327, kLambdaD = 0.5875618, kLambdaC = 0.6562725;  // um (Fraunhofer F, d, C)

[[noreturn]] void fail(plt_status code, const std::string& msg) { throw Error{code, msg}; }
}  // namespace

// ---------------------------------------------------------------------------
// Glass (paper silent; Abbe via Cauchy, Sellmeier as catalogued)
// ---------------------------------------------------------------------------
double Glass::index(double lambda_nm) const {
    const double l = lambda_nm * 1e-3, l2 = l * l;
    switch (model) {
        case kConst: return c[0];
        case kCauchy: return c[0] + c[1] / l2 + c[2] / (l2 * l2);
        case kAbbe: {
            double B = (c[0] - 1.0) / (c[1] * (1.0 / (kLambdaF * kLambdaF) - 1.0 / (kLambdaC * kLambdaC)));
            double A = c[0] - B / (kLambdaD * kLambdaD);
            return A + B / l2;
        }
        case kSellmeier: {
            double s = 1.0;
            for (int i = 0; i < 3; ++i) s += c[i] * l2 / (l2 - c[3 + i]);
            return std::sqrt(s);
        }
    }
    return NAN;
}

void Glass::device_form(int* gform, double g[6]) const {
    for (int i = 0; i < 6; ++i) g[i] = 0.0;
    switch (model) {
        case kConst: *gform = kCauchyForm; g[0] = c[0]; break;
        case kCauchy: *gform = kCauchyForm; g[0] = c[0]; g[1] = c[1]; g[2] = c[2]; break;
        case kAbbe: {
            double B = (c[0] - 1.0) / (c[1] * (1.0 / (kLambdaF * kLambdaF) - 1.0 / (kLambdaC * kLambdaC)));
            *gform = kCauchyForm; g[0] = c[0] - B / (kLambdaD * kLambdaD); g[1] = B; break;
        }
        case kSellmeier: *gform = kSellmeier; for (int i = 0; i < 6; ++i) g[i] = c[i]; break;
    }
}

// ---------------------------------------------------------------------------
// Parsing
// ---------------------------------------------------------------------------
namespace {

struct Row {
    double R, t, d; bool stop; Glass g; int line;
    bool asph = false; double k = 0, A[4] = {0, 0, 0, 0};
    double coat_n = 0, coat_d_um = 0;
};

bool parse_double(const std::string& s, double* v) {
    if (s.empty()) return false;
    char* end = nullptr;
    *v = std::strtod(s.c_str(), &end);
    return end && *end == '\0' && std::isfinite(*v);
}

std::vector<double> parse_list(const std::string& s, int line, const std::string& what) {
    std::vector<double> v;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) {
        double x;
        if (!parse_double(item, &x))
            fail(PLT_E_PARSE, "line " + std::to_string(line) + ": bad number '" + item + "' in " + what);
        v.push_back(x);
    }
    return v;
}

// Returns false for "stop".
bool parse_glass(const std::string& tok_in, const std::string* vd, int line, Glass* g) {
    std::string tok = tok_in;
    std::transform(tok.begin(), tok.end(), tok.begin(), [](unsigned char ch) { return std::tolower(ch); });
    *g = Glass{};
    if (tok == "air") return true;
    if (tok == "stop") return false;
    auto colon = tok.find(':');
    if (colon != std::string::npos) {
        std::string kind = tok.substr(0, colon);
        std::vector<double> v = parse_list(tok.substr(colon + 1), line, "glass '" + tok_in + "'");
        auto need = [&](size_t k) {
            if (v.size() < k)
                fail(PLT_E_PARSE, "line " + std::to_string(line) + ": glass '" + tok_in + "' needs " +
                                      std::to_string(k) + " coefficients");
        };
        if (kind == "n") { need(1); g->model = Glass::kConst; g->c[0] = v[0]; }
        else if (kind == "abbe") { need(2); g->model = Glass::kAbbe; g->c[0] = v[0]; g->c[1] = v[1]; }
        else if (kind == "cauchy") {
            need(1); g->model = Glass::kCauchy;
            for (size_t i = 0; i < 3; ++i) g->c[i] = i < v.size() ? v[i] : 0.0;
        } else if (kind == "sellmeier") {
            need(6); g->model = Glass::kSellmeier;
            for (int i = 0; i < 6; ++i) g->c[i] = v[i];
        } else fail(PLT_E_PARSE, "line " + std::to_string(line) + ": unknown glass kind '" + kind + "'");
        return true;
    }
    double nd;
    if (!parse_double(tok, &nd)) fail(PLT_E_PARSE, "line " + std::to_string(line) + ": bad glass '" + tok_in + "'");
    if (nd == 0.0) return false;    // Kolb: n_d = 0 marks the stop
    if (nd == 1.0) return true;     // air
    if (vd) {
        double v;
        if (!parse_double(*vd, &v)) fail(PLT_E_PARSE, "line " + std::to_string(line) + ": bad V_d '" + *vd + "'");
        g->model = Glass::kAbbe; g->c[0] = nd; g->c[1] = v;
    } else {
        g->model = Glass::kConst; g->c[0] = nd;
    }
    return true;
}

// --- minimal JSON reader (objects, arrays, strings, numbers, literals) -------
struct JVal {
    enum T { kNull, kBool, kNum, kStr, kArr, kObj } t = kNull;
    double num = 0; bool b = false; std::string str;
    std::vector<JVal> arr; std::vector<std::pair<std::string, JVal>> obj;
    const JVal* get(const std::string& k) const {
        for (auto& kv : obj) if (kv.first == k) return &kv.second;
        return nullptr;
    }
};

struct JParser {
    const char* p; const char* e;
    [[noreturn]] void err(const std::string& m) {
        fail(PLT_E_PARSE, "JSON: " + m + " at offset " + std::to_string(p - start));
    }
    const char* start;
    void ws() { while (p < e && std::isspace((unsigned char)*p)) ++p; }
    JVal value() {
        ws();
        if (p >= e) err("unexpected end");
        JVal v;
        if (*p == '{') {
            v.t = JVal::kObj; ++p; ws();
            if (p < e && *p == '}') { ++p; return v; }
            for (;;) {
                ws(); JVal k = value();
                if (k.t != JVal::kStr) err("object key must be a string");
                ws(); if (p >= e || *p != ':') err("expected ':'"); ++p;
                v.obj.emplace_back(k.str, value()); ws();
                if (p < e && *p == ',') { ++p; continue; }
                if (p < e && *p == '}') { ++p; return v; }
                err("expected ',' or '}'");
            }
        }
        if (*p == '[') {
            v.t = JVal::kArr; ++p; ws();
            if (p < e && *p == ']') { ++p; return v; }
            for (;;) {
                v.arr.push_back(value()); ws();
                if (p < e && *p == ',') { ++p; continue; }
                if (p < e && *p == ']') { ++p; return v; }
                err("expected ',' or ']'");
            }
        }
        if (*p == '"') {
            v.t = JVal::kStr; ++p;
            while (p < e && *p != '"') {
                if (*p == '\\' && p + 1 < e) { ++p; }
                v.str.push_back(*p++);
            }
            if (p >= e) err("unterminated string");
            ++p; return v;
        }
        if (!std::strncmp(p, "true", 4)) { p += 4; v.t = JVal::kBool; v.b = true; return v; }
        if (!std::strncmp(p, "false", 5)) { p += 5; v.t = JVal::kBool; return v; }
        if (!std::strncmp(p, "null", 4)) { p += 4; return v; }
        const char* q = p;
        while (q < e && (std::isdigit((unsigned char)*q) || *q == '-' || *q == '+' || *q == '.' || *q == 'e' || *q == 'E')) ++q;
        if (q == p) err("unexpected character");
        std::string s(p, q);
        if (!parse_double(s, &v.num)) err("bad number '" + s + "'");
        v.t = JVal::kNum; p = q; return v;
    }
};

std::vector<Row> rows_from_json(const std::string& text, std::string* name) {
    JParser jp{text.data(), text.data() + text.size(), text.data()};
    JVal doc = jp.value();
    if (doc.t != JVal::kObj) fail(PLT_E_PARSE, "JSON: top level must be an object");
    if (auto n = doc.get("name")) if (n->t == JVal::kStr) *name = n->str;
    auto s = doc.get("surfaces");
    if (!s || s->t != JVal::kArr) fail(PLT_E_PARSE, "JSON: missing 'surfaces' array");
    std::vector<Row> rows;
    int idx = 0;
    for (auto& it : s->arr) {
        ++idx;
        auto num = [&](const char* k) {
            auto v = it.get(k);
            if (!v || v->t != JVal::kNum) fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": missing number '" + k + "'");
            return v->num;
        };
        Row r{};
        r.R = num("radius_mm"); r.t = num("thickness_mm"); r.d = 2.0 * num("semi_aperture_mm"); r.line = idx;
        auto g = it.get("glass");
        std::string gs = g && g->t == JVal::kStr ? g->str : (g && g->t == JVal::kNum ? std::to_string(g->num) : "");
        if (gs.empty()) fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": missing 'glass'");
        r.stop = !parse_glass(gs, nullptr, idx, &r.g);
        if (auto co = it.get("coating")) {
            auto n = co->get("n"), l0 = co->get("lambda0_nm");
            if (co->t != JVal::kObj || !n || !l0 || n->t != JVal::kNum || l0->t != JVal::kNum)
                fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": 'coating' needs numbers 'n' and 'lambda0_nm'");
            r.coat_n = n->num;
            r.coat_d_um = l0->num * 1e-3 / (4.0 * n->num);
        }
        auto conic = it.get("conic");
        auto asp = it.get("aspheric");
        if (conic || asp) {
            r.asph = true;
            if (conic) {
                if (conic->t != JVal::kNum) fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": 'conic' must be a number");
                r.k = conic->num;
            }
            if (asp) {
                if (asp->t != JVal::kArr || asp->arr.size() > 4)
                    fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": 'aspheric' must be [A4, A6, A8, A10]");
                for (size_t i = 0; i < asp->arr.size(); ++i) {
                    if (asp->arr[i].t != JVal::kNum) fail(PLT_E_PARSE, "JSON surface " + std::to_string(idx) + ": bad aspheric coefficient");
                    r.A[i] = asp->arr[i].num;
                }
            }
        }
        rows.push_back(r);
    }
    return rows;
}

std::vector<Row> rows_from_table(const std::string& text, std::string* name) {
    std::vector<Row> rows;
    std::stringstream ss(text);
    std::string line;
    int ln = 0;
    while (std::getline(ss, line)) {
        ++ln;
        auto hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        std::stringstream ls(line);
        std::vector<std::string> tok;
        std::string t;
        while (ls >> t) tok.push_back(t);
        if (tok.empty()) continue;
        if (tok[0] == "name") { if (tok.size() > 1) *name = tok[1]; continue; }
        Row r{};
        r.line = ln;
        for (;;) {   // optional trailing 'asph:k,A4,A6,A8,A10' and 'coat:n_c,lambda0_nm' (any order)
            std::string last = tok.back();
            std::transform(last.begin(), last.end(), last.begin(), [](unsigned char ch) { return std::tolower(ch); });
            if (tok.size() > 4 && last.rfind("asph:", 0) == 0) {
                std::vector<double> v = parse_list(last.substr(5), ln, "asph");
                if (v.empty() || v.size() > 5) fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": asph needs 1 to 5 numbers (k,A4,A6,A8,A10)");
                r.asph = true;
                r.k = v[0];
                for (size_t i = 1; i < v.size(); ++i) r.A[i - 1] = v[i];
                tok.pop_back();
            } else if (tok.size() > 4 && last.rfind("coat:", 0) == 0) {
                std::vector<double> v = parse_list(last.substr(5), ln, "coat");
                if (v.size() != 2 || !(v[0] > 1.0) || !(v[1] > 0.0))
                    fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": coat needs 'coat:n_c,lambda0_nm' with n_c > 1, lambda0 > 0");
                r.coat_n = v[0];
                r.coat_d_um = v[1] * 1e-3 / (4.0 * v[0]);
                tok.pop_back();
            } else {
                break;
            }
        }
        if (tok.size() < 4 || tok.size() > 5)
            fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": expected 'radius thickness glass aperture_diameter [V_d] [asph:k,A4,...]'");
        if (!parse_double(tok[0], &r.R)) fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": bad radius '" + tok[0] + "'");
        if (!parse_double(tok[1], &r.t)) fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": bad thickness '" + tok[1] + "'");
        if (!parse_double(tok[3], &r.d)) fail(PLT_E_PARSE, "line " + std::to_string(ln) + ": bad aperture '" + tok[3] + "'");
        r.stop = !parse_glass(tok[2], tok.size() == 5 ? &tok[4] : nullptr, ln, &r.g);
        rows.push_back(r);
    }
    return rows;
}

}  // namespace

plt_lens* parse_lens(const char* text, size_t len, const plt_lens_opts* opts) {
    std::string s(text, len);
    std::string name = "lens";
    size_t first = s.find_first_not_of(" \t\r\n");
    std::vector<Row> rows = (first != std::string::npos && s[first] == '{') ? rows_from_json(s, &name)
                                                                           : rows_from_table(s, &name);
    if (rows.empty()) fail(PLT_E_VALIDATION, "no surfaces");
    auto L = std::make_unique<plt_lens>();
    L->name = name;
    double z = 0.0;
    Glass prev;  // air before surface 1
    int nstop = 0;
    for (size_t k = 0; k < rows.size(); ++k) {
        const Row& r = rows[k];
        const std::string where = "surface " + std::to_string(k + 1) + " (line " + std::to_string(r.line) + ")";
        if (!(r.d > 0)) fail(PLT_E_VALIDATION, where + ": clear aperture must be > 0");
        if (k + 1 < rows.size() && !(r.t > 0))
            fail(PLT_E_VALIDATION, where + ": non-increasing axial position (thickness must be > 0)");
        if (r.t < 0) fail(PLT_E_VALIDATION, where + ": negative thickness");
        Surface sf;
        sf.z = z;
        sf.a = 0.5 * r.d;
        sf.stop = r.stop;
        sf.R = r.stop ? 0.0 : r.R;
        sf.before = prev;
        sf.after = r.stop ? prev : r.g;
        if (r.coat_n > 0.0 && !r.stop) {
            const bool air_side = (sf.before.model == Glass::kConst && sf.before.c[0] == 1.0) ||
                                  (sf.after.model == Glass::kConst && sf.after.c[0] == 1.0);
            if (!air_side) fail(PLT_E_VALIDATION, where + ": coatings are modelled on air-glass surfaces only");
            sf.coat_n = r.coat_n;
            sf.coat_d_um = r.coat_d_um;
        }
        if (r.asph && !r.stop) {
            sf.asph = true;
            sf.k = r.k;
            for (int i = 0; i < 4; ++i) sf.A[i] = r.A[i];
            const double c = sf.R == 0.0 ? 0.0 : 1.0 / sf.R;
            if (1.0 - (1.0 + sf.k) * c * c * sf.a * sf.a < 0.0)
                fail(PLT_E_VALIDATION, where + ": conic surface undefined inside the clear aperture");
        } else if (!r.stop && sf.R != 0.0 && std::fabs(sf.R) < sf.a)
            fail(PLT_E_VALIDATION, where + ": |radius| < clear semi-aperture (cap would not span the aperture)");
        if (r.stop) { ++nstop; L->stop_index = (int)k; }
        else ++L->n_optical;
        for (double lam = 380.0; lam <= 780.0; lam += 20.0) {
            double n = sf.after.index(lam);
            if (!(n >= 1.0)) fail(PLT_E_VALIDATION, where + ": refractive index < 1 (or NaN) in [380,780] nm");
        }
        L->surf.push_back(sf);
        prev = sf.after;
        z += r.t;
    }
    if (nstop > 1) fail(PLT_E_VALIDATION, "more than one aperture stop");
    if (L->n_optical == 0) fail(PLT_E_VALIDATION, "no optical surface");
    plt_lens_opts o{};
    o.input_plane_z_mm = -5.0;
    o.sensor_z_mm = NAN;
    o.backward_exit_z_mm = -5.0;
    o.lambda_ref_nm = 587.5618;
    if (opts) o = *opts;
    if (!(o.lambda_ref_nm >= 380.0 && o.lambda_ref_nm <= 780.0)) fail(PLT_E_INVALID_ARG, "lambda_ref_nm outside [380,780]");
    if (o.sensor_w_mm < 0 || o.sensor_h_mm < 0 || o.housing_radius_mm < 0)
        fail(PLT_E_INVALID_ARG, "negative sensor size or housing radius");
    L->opts = o;
    if (std::isnan(o.sensor_z_mm)) {
        double M[4];
        lens_abcd(*L, o.lambda_ref_nm, M);
        if (M[2] == 0.0) fail(PLT_E_VALIDATION, "afocal lens: sensor_z_mm must be given explicitly");
        L->sensor_z = L->surf.back().z - M[0] / M[2];   // paraxial focus = last vertex + BFL
    } else {
        L->sensor_z = o.sensor_z_mm;
    }
    return L.release();
}

// ---------------------------------------------------------------------------
// ABCD: refraction [[1,0],[(n1-n2)/(n2 R), n1/n2]],
// translation [[1,d],[0,1]]; M from just before the first vertex to just after the last.
// ---------------------------------------------------------------------------
void lens_abcd(const plt_lens& L, double lambda_nm, double M[4]) {
    double a = 1, b = 0, c = 0, d = 1;  // row-major [[a,b],[c,d]]
    for (size_t k = 0; k < L.surf.size(); ++k) {
        const Surface& s = L.surf[k];
        if (k > 0) {  // translation T = [[1,t],[0,1]] : M <- T M
            double t = s.z - L.surf[k - 1].z;
            a += t * c; b += t * d;
        }
        double n1 = s.before.index(lambda_nm), n2 = s.after.index(lambda_nm);
        double p = (s.R == 0.0) ? 0.0 : (n1 - n2) / (n2 * s.R);
        double q = n1 / n2;
        double c2 = p * a + q * c, d2 = p * b + q * d;   // [[1,0],[p,q]] M
        c = c2; d = d2;
    }
    M[0] = a; M[1] = b; M[2] = c; M[3] = d;
}

// ---------------------------------------------------------------------------
// Paraxial pupils: the aperture stop imaged through the rear group (exit pupil: distance
// s' = -B/D behind the last vertex, magnification 1/D in air) and through the front group
// (entrance pupil: object plane at z_first + B/A conjugate to the stop, magnification A).
// ---------------------------------------------------------------------------
void lens_pupils(const plt_lens& L, double lambda_nm, double out[4]) {
    if (L.stop_index < 0) fail(PLT_E_VALIDATION, "lens has no aperture stop");
    const Surface& st = L.surf[(size_t)L.stop_index];
    // group matrix [[a,b],[c,d]] from plane z0 through surfaces [i0, i1) (stops skipped)
    auto group = [&](size_t i0, size_t i1, double z0, double* zl) {
        double a = 1, b = 0, c = 0, d = 1, z = z0;
        for (size_t k = i0; k < i1; ++k) {
            const Surface& s = L.surf[k];
            if (s.stop) continue;
            const double t = s.z - z;
            a += t * c; b += t * d;
            const double n1 = s.before.index(lambda_nm), n2 = s.after.index(lambda_nm);
            const double p = s.R == 0.0 ? 0.0 : (n1 - n2) / (n2 * s.R), q = n1 / n2;
            const double c2 = p * a + q * c, d2 = p * b + q * d;
            c = c2; d = d2;
            z = s.z;
        }
        *zl = z;
        return std::array<double, 4>{a, b, c, d};
    };
    const size_t k = (size_t)L.stop_index;
    bool rear = false, front = false;
    for (size_t i = k + 1; i < L.surf.size(); ++i) rear |= !L.surf[i].stop;
    for (size_t i = 0; i < k; ++i) front |= !L.surf[i].stop;
    if (front) {
        double zl;
        size_t first = 0;
        while (L.surf[first].stop) ++first;
        auto N = group(first, k, L.surf[first].z, &zl);
        const double t = st.z - zl;                 // translate to the stop plane
        N[0] += t * N[2]; N[1] += t * N[3];
        out[0] = L.surf[first].z + N[1] / N[0];
        out[1] = st.a / std::fabs(N[0]);
    } else {
        out[0] = st.z; out[1] = st.a;
    }
    if (rear) {
        double zl;
        auto M = group(k + 1, L.surf.size(), st.z, &zl);
        out[2] = zl - M[1] / M[3];
        out[3] = st.a / std::fabs(M[3]);
    } else {
        out[2] = st.z; out[3] = st.a;
    }
}

// ---------------------------------------------------------------------------
// Path programs (Eq. 3-4; SURVEY A9 sentinel LSB-first id)
// ---------------------------------------------------------------------------
namespace {

std::vector<Surface> traversal_frame(const plt_lens& L, int dir, double* zS) {
    *zS = L.surf.back().z;
    if (dir == PLT_FORWARD) return L.surf;
    std::vector<Surface> m;  // mirror: z' = zS - z, R' = -R, order reversed, before/after swapped (C0)
    for (auto it = L.surf.rbegin(); it != L.surf.rend(); ++it) {
        Surface s = *it;
        s.z = *zS - it->z;
        s.R = it->R == 0.0 ? 0.0 : -it->R;
        for (int i = 0; i < 4; ++i) s.A[i] = -it->A[i];   // mirrored sag is -sag
        s.before = it->after;
        s.after = it->before;
        m.push_back(s);
    }
    return m;
}

template <typename T>
void fill_step(Step<T>* st, const Surface& s, int kind, int is_R, int dir, const Glass& far) {
    st->z = (T)s.z;
    st->R = (T)s.R;
    st->twoR = (T)(2.0 * s.R);
    st->invR = s.R == 0.0 ? (T)0 : (T)(1.0 / s.R);
    st->a2 = (T)(s.a * s.a);
    st->band_a = (T)(2.0 * s.a * kTraceBandEdge);
    st->sdir = (T)dir;
    st->kind = kind;
    st->is_R = is_R;
    st->pad = 0;
    st->asph[0] = (T)s.k;
    for (int i = 0; i < 4; ++i) st->asph[1 + i] = (T)s.A[i];
    st->coat_n = (T)s.coat_n;
    st->coat_kpi = (T)(4.0 * s.coat_n * s.coat_d_um);
    double g[6];
    far.device_form(&st->gform, g);
    for (int i = 0; i < 6; ++i) st->g[i] = (T)g[i];
}

}  // namespace

std::shared_ptr<CompiledPath> compile_path(const plt_lens& L, uint64_t path_id, int dir) {
    {
        std::lock_guard<std::mutex> g(L.mu);
        auto it = L.cache.find({path_id, dir});
        if (it != L.cache.end()) return it->second;
    }
    if (path_id < 2) fail(PLT_E_INVALID_ARG, "path id must be >= 2 (sentinel bit plus at least one interaction)");
    int K = 63;
    while (!((path_id >> K) & 1ull)) --K;
    double zS;
    std::vector<Surface> fr = traversal_frame(L, dir, &zS);
    auto cp = std::make_shared<CompiledPath>();
    std::memset(&cp->pf, 0, sizeof cp->pf);
    std::memset(&cp->pd, 0, sizeof cp->pd);
    int s = 0, d = +1, k = 0, ns = 0;
    const int S = (int)fr.size();
    while (s >= 0 && s < S) {
        if (ns >= kMaxSteps) fail(PLT_E_INVALID_ARG, "path needs more than " + std::to_string(kMaxSteps) + " surface steps");
        const Surface& sf = fr[s];
        if (sf.stop) {
            fill_step(&cp->pf.st[ns], sf, kStop, 0, d, sf.after);
            fill_step(&cp->pd.st[ns], sf, kStop, 0, d, sf.after);
            ++ns;
            s += d;
            continue;
        }
        if (k >= K) fail(PLT_E_INVALID_ARG, "path id " + std::to_string(path_id) + " is inconsistent with the lens (interactions exhausted inside the lens)");
        const int isR = (int)((path_id >> k) & 1ull);
        const Glass& far = d > 0 ? sf.after : sf.before;
        const int kind = sf.asph ? kAsphere : (sf.R == 0.0 ? kPlane : kSphere);
        fill_step(&cp->pf.st[ns], sf, kind, isR, d, far);
        fill_step(&cp->pd.st[ns], sf, kind, isR, d, far);
        ++ns;
        ++k;
        if (isR) d = -d;
        s += d;
    }
    if (d < 0 || k != K)
        fail(PLT_E_INVALID_ARG, "path id " + std::to_string(path_id) + " is inconsistent with the lens (" +
                                    (d < 0 ? "exits through the front" : "interactions left over") + ")");
    const double z_out = dir == PLT_FORWARD ? L.sensor_z : zS - L.opts.backward_exit_z_mm;
    const bool rect = dir == PLT_FORWARD && L.opts.sensor_w_mm > 0 && L.opts.sensor_h_mm > 0;
    const double H = L.opts.housing_radius_mm;
    // block-level compaction point: right after the (first) stop crossing, else mid-path
    int split = ns / 2;
    for (int i = 0; i < ns; ++i)
        if (cp->pf.st[i].kind == kStop) { if (i + 1 < ns && i > 0) split = i + 1; break; }
    // backward (camera) queries start on the sensor side, where the rear elements vignette
    // most rays within the first steps (the 24 mm camera keeps 26 % after two steps, 10 % at
    // the stop): compacting two steps before the stop measured 6 % faster there
    if (dir == PLT_BACKWARD && split - 2 >= 2) split -= 2;
    if (const char* e = std::getenv("PLT_TRACE_SPLIT_DELTA")) {   // developer tuning knob
        const int v = split + std::atoi(e);
        if (v > 0 && v < ns) split = v;
    }
    auto fill_prog = [&](auto& P) {
        using T = std::remove_reference_t<decltype(P.z_out)>;
        P.n_steps = ns;
        P.split = split;
        P.band_h = (T)(2.0 * H * kTraceBandEdge);
        P.flip = dir == PLT_BACKWARD;
        P.has_rect = rect;
        P.has_housing = H > 0;
        P.has_asph = 0;
        for (int i = 0; i < ns; ++i) P.has_asph |= P.st[i].kind == kAsphere || P.st[i].coat_n > 0;
        P.z_out = (T)z_out;
        P.z_mirror = (T)zS;
        P.housing = (T)H;
        P.housing2 = (T)(H * H);
        P.rect_hw = (T)(0.5 * L.opts.sensor_w_mm);
        P.rect_hh = (T)(0.5 * L.opts.sensor_h_mm);
        P.rect_cx = 0;
        P.rect_cy = 0;
    };
    fill_prog(cp->pf);
    fill_prog(cp->pd);
    std::lock_guard<std::mutex> g(L.mu);
    L.cache[{path_id, dir}] = cp;
    return cp;
}

// ---------------------------------------------------------------------------
// Ghost enumeration (§4.2; ids P:193)
// ---------------------------------------------------------------------------
namespace {
// Normal-incidence throughput of a path at lambda (R0 = ((n1-n2)/(n1+n2))^2 per interface).
double normal_incidence_throughput(const plt_lens& L, uint64_t id, double lam) {
    std::vector<const Surface*> opt;
    for (auto& s : L.surf) if (!s.stop) opt.push_back(&s);
    int K = 63;
    while (!((id >> K) & 1ull)) --K;
    int s = 0, d = 1;
    double ncur = 1.0, I = 1.0;
    for (int k = 0; k < K; ++k) {
        if (s < 0 || s >= (int)opt.size()) return -1.0;
        const Surface& sf = *opt[s];
        double n2 = (d > 0 ? sf.after : sf.before).index(lam);
        double r0;
        if (sf.coat_n > 0.0) {   // thin film at normal incidence (as the trace's Airy formula)
            const double nc = sf.coat_n, a = (ncur - nc) / (ncur + nc), b = (nc - n2) / (nc + n2);
            const double cb = std::cos(4.0 * 3.14159265358979323846 * nc * sf.coat_d_um / (lam * 1e-3));
            r0 = (a * a + b * b + 2 * a * b * cb) / (1 + a * a * b * b + 2 * a * b * cb);
        } else {
            r0 = (ncur - n2) / (ncur + n2);
            r0 *= r0;
        }
        if ((id >> k) & 1ull) { I *= r0; d = -d; }
        else { I *= 1.0 - r0; ncur = n2; }
        s += d;
    }
    return I;
}
}  // namespace

std::vector<std::pair<uint64_t, std::pair<int, int>>> enumerate_ghosts(const plt_lens& L, int max_bounces,
                                                                       double min_throughput) {
    const int m = L.n_optical;
    std::vector<std::pair<uint64_t, std::pair<int, int>>> out;
    out.push_back({1ull << m, {0, 0}});
    auto keep = [&](uint64_t id) {
        return !(min_throughput > 0.0 && normal_incidence_throughput(L, id, L.opts.lambda_ref_nm) < min_throughput);
    };
    if (max_bounces >= 2) {
        for (int i = 2; i <= m; ++i)
            for (int j = 1; j < i; ++j) {
                const int K = m + 2 * (i - j);
                if (K > 63) continue;
                uint64_t id = (1ull << K) + (1ull << (i - 1)) + (1ull << (2 * i - j - 1));
                if (keep(id)) out.push_back({id, {i, j}});
            }
    }
    if (max_bounces >= 4) {   // reflect at i, back to j, forward to k, back to l (NEXT-4)
        for (int j = 1; j < m; ++j)
            for (int i = j + 1; i <= m; ++i)
                for (int k = j + 1; k <= m; ++k)
                    for (int l = 1; l < k; ++l) {
                        const int K = m + 2 * (i - j) + 2 * (k - l);
                        if (K > 63) continue;
                        const int r1 = i - 1, r2 = r1 + (i - j), r3 = r2 + (k - j), r4 = r3 + (k - l);
                        const uint64_t id = (1ull << K) | (1ull << r1) | (1ull << r2) | (1ull << r3) | (1ull << r4);
                        if (keep(id)) out.push_back({id, {i, j}});
                    }
    }
    std::sort(out.begin(), out.end());
    return out;
}

}  // namespace plt
