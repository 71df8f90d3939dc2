// Native codec for the bulk of the reference's scene documents (reference
// sceneio.py:57-239): the "masses" and "springs" arrays, which are all but a
// few hundred bytes of a lattice document (1.7 GB of text at 10M springs).
//
// Rendering writes exactly the text json.dumps(doc, indent=2) produces for
// those arrays (sceneio.py:57-75): the same key order, 2-space indentation,
// one vector component per line, and Python's float repr -- the shortest
// digit string that round-trips (std::to_chars, Ryu) laid out by repr's
// rule: positional notation when the decimal exponent is in [-4, 16), else
// d.ddde+XX with at least two exponent digits.  tests/test_sceneio_native.py
// compares it with repr() on millions of doubles and with the reference's
// render_scene on whole documents.
//
// Parsing is a strict fast path: it reads the top-level object, returns the
// raw text span of every other top-level value (the host decodes those few
// with json.loads) and decodes the two arrays into columns.  Anything outside
// the plain case -- a syntax error, an unknown/missing/duplicate field, a
// wrong type, a non-contiguous id, an escape sequence in a string, an
// integer beyond int64, NaN/Infinity literals, non-ASCII text -- returns
// SS_EFALLBACK and the host runs the reference-exact Python parser, which
// then reports the precise error.  So every accepted document yields
// exactly what the Python path yields (numbers by std::from_chars, correctly
// rounded like Python's float()).
#include <omp.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "springsim_b200.h"

namespace {

// ------------------------------------------------------------------ render

// Python repr(float) of a finite double into p; returns the end.
char *put_double(char *p, double v) {
    if (v == 0.0) {
        if (std::signbit(v)) *p++ = '-';
        std::memcpy(p, "0.0", 3);
        return p + 3;
    }
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    const char *q = buf;
    if (*q == '-') {
        *p++ = '-';
        ++q;
    }
    char dig[24];
    int nd = 0;
    for (; q < r.ptr && *q != 'e'; ++q)
        if (*q != '.') dig[nd++] = *q;
    int e10 = 0;                               // "e+XX" / "e-XX" (buf is not NUL-terminated)
    const char *ep = q + 1;
    if (ep < r.ptr && *ep == '+') ++ep;
    std::from_chars(ep, r.ptr, e10);
    const int decpt = e10 + 1;
    if (decpt <= -4 || decpt > 16) {           // d[.ddd]e+XX
        *p++ = dig[0];
        if (nd > 1) {
            *p++ = '.';
            std::memcpy(p, dig + 1, nd - 1);
            p += nd - 1;
        }
        *p++ = 'e';
        *p++ = e10 < 0 ? '-' : '+';
        const int a = e10 < 0 ? -e10 : e10;
        if (a < 10) *p++ = '0';
        p = std::to_chars(p, p + 4, a).ptr;
    } else if (decpt <= 0) {                   // 0.000ddd
        *p++ = '0';
        *p++ = '.';
        for (int z = 0; z < -decpt; ++z) *p++ = '0';
        std::memcpy(p, dig, nd);
        p += nd;
    } else if (decpt >= nd) {                  // ddd000.0
        std::memcpy(p, dig, nd);
        p += nd;
        for (int z = nd; z < decpt; ++z) *p++ = '0';
        *p++ = '.';
        *p++ = '0';
    } else {                                   // dd.ddd
        std::memcpy(p, dig, decpt);
        p += decpt;
        *p++ = '.';
        std::memcpy(p, dig + decpt, nd - decpt);
        p += nd - decpt;
    }
    return p;
}

char *put_str(char *p, const char *s) {
    const size_t n = std::strlen(s);
    std::memcpy(p, s, n);
    return p + n;
}

char *put_i64(char *p, int64_t v) { return std::to_chars(p, p + 24, v).ptr; }

char *put_vec(char *p, const char *key, const double *c) {
    p = put_str(p, key);                       // '      "x": [\n'
    for (int i = 0; i < 3; ++i) {
        p = put_str(p, "        ");
        p = put_double(p, c[i]);
        p = put_str(p, i < 2 ? ",\n" : "\n");
    }
    return put_str(p, "      ]");
}

// Upper bounds of one entry's text (floats <= 24 chars, ints <= 20).
constexpr size_t kMassMax = 420;
constexpr size_t kSpringFixed = 160;

bool all_finite(const double *a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!std::isfinite(a[i])) return false;
    return true;
}

// Render entries [0, n) in parallel blocks (entries joined by ",\n").
template <typename One>
std::vector<std::string> render_parts(int64_t n, size_t per_entry, One one) {
    const int64_t block = 1 << 14;
    const int64_t nb = (n + block - 1) / block;
    std::vector<std::string> parts((size_t)nb);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t i0 = b * block, i1 = std::min(n, i0 + block);
        std::string &s = parts[(size_t)b];
        s.resize((size_t)(i1 - i0) * per_entry);
        char *p = s.data();
        for (int64_t i = i0; i < i1; ++i) {
            if (i) p = put_str(p, ",\n");
            p = one(p, i);
        }
        s.resize((size_t)(p - s.data()));
    }
    return parts;
}

// The pieces in order, into one malloc'd buffer (parallel copies).
int concat(const std::vector<const std::string *> &pieces, char **out, int64_t *len) {
    std::vector<size_t> off(pieces.size() + 1, 0);
    for (size_t i = 0; i < pieces.size(); ++i) off[i + 1] = off[i] + pieces[i]->size();
    char *buf = static_cast<char *>(std::malloc(off.back() + 1));
    if (!buf) return SS_ENOMEM;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < (int64_t)pieces.size(); ++i)
        std::memcpy(buf + off[i], pieces[i]->data(), pieces[i]->size());
    *out = buf;
    *len = (int64_t)off.back();
    return SS_OK;
}

template <typename One>
int render_blocks(int64_t n, size_t per_entry, One one, char **out, int64_t *len) {
    *out = nullptr;
    *len = 0;
    const auto parts = render_parts(n, per_entry, one);
    std::vector<const std::string *> pieces;
    for (const auto &p : parts) pieces.push_back(&p);
    return concat(pieces, out, len);
}

// ------------------------------------------------------------------ parse

struct Doc {
    std::vector<std::string> keys;             // top-level keys, document order
    std::vector<int64_t> off, span;            // their values' raw text
    std::vector<double> m, x, v, f, k, l0;
    std::vector<uint8_t> fixed;
    std::vector<int64_t> si, sj;
    std::vector<int32_t> group;                // index into labels, -1 null
    std::vector<std::string> labels;           // distinct spring group strings, first-appearance order
};

struct Reader {
    const char *s;
    const char *e;
    bool ok = true;

    void ws() {
        while (s < e && (*s == ' ' || *s == '\n' || *s == '\t' || *s == '\r')) ++s;
    }
    bool lit(char c) {
        ws();
        if (s < e && *s == c) {
            ++s;
            return true;
        }
        return false;
    }
    void need(char c) {
        if (!lit(c)) ok = false;
    }
    // a plain string (no escapes, no control characters)
    bool str(const char *&a, size_t &n) {
        ws();
        if (s >= e || *s != '"') return ok = false;
        a = ++s;
        while (s < e && *s != '"') {
            if (*s == '\\' || (unsigned char)*s < 0x20 || (unsigned char)*s >= 0x80) return ok = false;
            ++s;
        }
        if (s >= e) return ok = false;
        n = (size_t)(s - a);
        ++s;
        return true;
    }
    // a JSON number token; is_int: no fraction/exponent
    bool num_token(const char *&a, const char *&b, bool &is_int) {
        ws();
        a = s;
        const char *p = s;
        if (p < e && *p == '-') ++p;
        if (p >= e) return ok = false;
        if (*p == '0') {
            ++p;
        } else if (*p >= '1' && *p <= '9') {
            while (p < e && *p >= '0' && *p <= '9') ++p;
        } else {
            return ok = false;
        }
        is_int = true;
        if (p < e && *p == '.') {
            ++p;
            if (p >= e || *p < '0' || *p > '9') return ok = false;
            while (p < e && *p >= '0' && *p <= '9') ++p;
            is_int = false;
        }
        if (p < e && (*p == 'e' || *p == 'E')) {
            ++p;
            if (p < e && (*p == '+' || *p == '-')) ++p;
            if (p >= e || *p < '0' || *p > '9') return ok = false;
            while (p < e && *p >= '0' && *p <= '9') ++p;
            is_int = false;
        }
        b = p;
        s = p;
        return true;
    }
    bool number(double &out) {                 // "number": int or float -> double
        const char *a, *b;
        bool is_int;
        if (!num_token(a, b, is_int)) return false;
        const auto r = std::from_chars(a, b, out);
        if (r.ec != std::errc() || r.ptr != b || !std::isfinite(out)) return ok = false;
        return true;
    }
    bool integer(int64_t &out) {               // "int": integer token within int64
        const char *a, *b;
        bool is_int;
        if (!num_token(a, b, is_int) || !is_int) return ok = false;
        const auto r = std::from_chars(a, b, out);
        if (r.ec != std::errc() || r.ptr != b) return ok = false;
        return true;
    }
    bool boolean(bool &out) {
        ws();
        if (e - s >= 4 && std::memcmp(s, "true", 4) == 0) {
            s += 4;
            out = true;
            return true;
        }
        if (e - s >= 5 && std::memcmp(s, "false", 5) == 0) {
            s += 5;
            out = false;
            return true;
        }
        return ok = false;
    }
    bool null() {
        ws();
        if (e - s >= 4 && std::memcmp(s, "null", 4) == 0) {
            s += 4;
            return true;
        }
        return false;
    }
    bool vec3(double *c) {
        need('[');
        for (int i = 0; ok && i < 3; ++i) {
            if (i) need(',');
            if (ok) number(c[i]);
        }
        need(']');
        return ok;
    }
    // skip any JSON value (syntax-checked; strings may hold escapes)
    void skip() {
        ws();
        if (s >= e) {
            ok = false;
            return;
        }
        const char c = *s;
        if (c == '{' || c == '[') {
            const char close = c == '{' ? '}' : ']';
            ++s;
            if (lit(close)) return;
            do {
                if (c == '{') {
                    skip_string();
                    need(':');
                }
                if (ok) skip();
            } while (ok && lit(','));
            need(close);
        } else if (c == '"') {
            skip_string();
        } else if (c == 't' || c == 'f') {
            bool b;
            boolean(b);
        } else if (c == 'n') {
            if (!null()) ok = false;
        } else {
            const char *a, *b;
            bool i;
            num_token(a, b, i);
        }
    }
    void skip_string() {
        ws();
        if (s >= e || *s != '"') {
            ok = false;
            return;
        }
        ++s;
        while (s < e && *s != '"') {
            if ((unsigned char)*s < 0x20 || (unsigned char)*s >= 0x80) {
                ok = false;
                return;
            }
            if (*s == '\\') {
                ++s;
                if (s >= e) break;
                if (*s == 'u') {
                    for (int h = 0; h < 4; ++h) {
                        ++s;
                        if (s >= e || !std::isxdigit((unsigned char)*s)) {
                            ok = false;
                            return;
                        }
                    }
                } else if (!std::strchr("\"\\/bfnrt", *s)) {
                    ok = false;
                    return;
                }
            }
            ++s;
        }
        if (s >= e) {
            ok = false;
            return;
        }
        ++s;
    }
};

bool key_is(const char *a, size_t n, const char *k) { return std::strlen(k) == n && std::memcmp(a, k, n) == 0; }

// One mass object; fields of _MASS (sceneio.py:139-144), each at most once.
bool read_mass(Reader &r, Doc &d, int64_t idx) {
    double m = 0, x[3], v[3] = {0, 0, 0}, f[3] = {0, 0, 0};
    bool fixed = false, has_m = false, has_x = false;
    unsigned seen = 0;
    r.need('{');
    if (r.lit('}')) return false;              // missing required fields: the slow path words it
    do {
        const char *a;
        size_t n;
        if (!r.str(a, n)) return false;
        r.need(':');
        unsigned bit;
        if (key_is(a, n, "id")) {
            bit = 1;
            int64_t id;
            if (!r.integer(id) || id != idx) return false;
        } else if (key_is(a, n, "m")) {
            bit = 2;
            has_m = r.number(m);
        } else if (key_is(a, n, "x")) {
            bit = 4;
            has_x = r.vec3(x);
        } else if (key_is(a, n, "v")) {
            bit = 8;
            r.vec3(v);
        } else if (key_is(a, n, "f_ext")) {
            bit = 16;
            r.vec3(f);
        } else if (key_is(a, n, "fixed")) {
            bit = 32;
            r.boolean(fixed);
        } else {
            return false;
        }
        if (!r.ok || (seen & bit)) return false;
        seen |= bit;
    } while (r.lit(','));
    r.need('}');
    if (!r.ok || !has_m || !has_x) return false;
    d.m.push_back(m);
    d.x.insert(d.x.end(), x, x + 3);
    d.v.insert(d.v.end(), v, v + 3);
    d.f.insert(d.f.end(), f, f + 3);
    d.fixed.push_back(fixed ? 1 : 0);
    return true;
}

// One spring object; fields of _SPRING (sceneio.py:146-149).
bool read_spring(Reader &r, Doc &d, int64_t idx) {
    int64_t i = 0, j = 0;
    double k = 0, l0 = 0;
    int32_t g = -1;
    unsigned seen = 0;
    r.need('{');
    if (r.lit('}')) return false;
    do {
        const char *a;
        size_t n;
        if (!r.str(a, n)) return false;
        r.need(':');
        unsigned bit;
        if (key_is(a, n, "id")) {
            bit = 1;
            int64_t id;
            if (!r.integer(id) || id != idx) return false;
        } else if (key_is(a, n, "i")) {
            bit = 2;
            r.integer(i);
        } else if (key_is(a, n, "j")) {
            bit = 4;
            r.integer(j);
        } else if (key_is(a, n, "k")) {
            bit = 8;
            r.number(k);
        } else if (key_is(a, n, "l0")) {
            bit = 16;
            r.number(l0);
        } else if (key_is(a, n, "group")) {
            bit = 32;
            if (!r.null()) {
                const char *ga;
                size_t gn;
                if (!r.str(ga, gn)) return false;
                std::string lab(ga, gn);
                auto it = std::find(d.labels.begin(), d.labels.end(), lab);
                if (it == d.labels.end()) {
                    d.labels.push_back(lab);
                    g = (int32_t)d.labels.size() - 1;
                } else {
                    g = (int32_t)(it - d.labels.begin());
                }
            }
        } else {
            return false;
        }
        if (!r.ok || (seen & bit)) return false;
        seen |= bit;
    } while (r.lit(','));
    r.need('}');
    if (!r.ok || (seen & 30u) != 30u) return false;          // i, j, k, l0 required
    d.si.push_back(i);
    d.sj.push_back(j);
    d.k.push_back(k);
    d.l0.push_back(l0);
    d.group.push_back(g);
    return true;
}

template <typename ReadOne>
bool read_array(Reader &r, ReadOne one) {
    r.need('[');
    if (!r.ok) return false;
    if (r.lit(']')) return true;
    int64_t idx = 0;
    do {
        if (!one(idx++)) return false;
    } while (r.lit(','));
    r.need(']');
    return r.ok;
}

}  // namespace

struct ss_doc : Doc {};

namespace {

// One "masses" / "springs" entry at indent 4 (the text json.dumps writes).
auto mass_entry(const double *m, const double *x, const double *v, const double *f, const uint8_t *fixed) {
    return [=](char *p, int64_t i) {
        p = put_str(p, "    {\n      \"id\": ");
        p = put_i64(p, i);
        p = put_str(p, ",\n      \"m\": ");
        p = put_double(p, m[i]);
        p = put_str(p, ",\n");
        p = put_vec(p, "      \"x\": [\n", x + 3 * i);
        p = put_str(p, ",\n");
        p = put_vec(p, "      \"v\": [\n", v + 3 * i);
        p = put_str(p, ",\n");
        p = put_vec(p, "      \"f_ext\": [\n", f + 3 * i);
        return put_str(p, fixed[i] ? ",\n      \"fixed\": true\n    }" : ",\n      \"fixed\": false\n    }");
    };
}

auto spring_entry(const int64_t *si, const int64_t *sj, const double *k, const double *l0, const int32_t *group,
                  const char *const *labels) {
    return [=](char *p, int64_t s) {
        p = put_str(p, "    {\n      \"id\": ");
        p = put_i64(p, s);
        p = put_str(p, ",\n      \"i\": ");
        p = put_i64(p, si[s]);
        p = put_str(p, ",\n      \"j\": ");
        p = put_i64(p, sj[s]);
        p = put_str(p, ",\n      \"k\": ");
        p = put_double(p, k[s]);
        p = put_str(p, ",\n      \"l0\": ");
        p = put_double(p, l0[s]);
        p = put_str(p, ",\n      \"group\": ");
        p = put_str(p, group && group[s] >= 0 ? labels[group[s]] : "null");
        return put_str(p, "\n    }");
    };
}

// Argument checks shared by the renderers: SS_EINVAL, SS_EFALLBACK for a
// non-finite value (json.dumps(allow_nan=False) raises: the host words it),
// else SS_OK with the longest group label in *longest.
int check_masses(int64_t n, const double *m, const double *x, const double *v, const double *f, const uint8_t *fixed) {
    if (n < 0 || (n && (!m || !x || !v || !f || !fixed))) return SS_EINVAL;
    if (!all_finite(m, n) || !all_finite(x, 3 * n) || !all_finite(v, 3 * n) || !all_finite(f, 3 * n))
        return SS_EFALLBACK;
    return SS_OK;
}

int check_springs(int64_t n, const int64_t *si, const int64_t *sj, const double *k, const double *l0,
                  const int32_t *group, const char *const *labels, int32_t n_labels, size_t *longest) {
    if (n < 0 || (n && (!si || !sj || !k || !l0)) || n_labels < 0 || (n_labels && !labels)) return SS_EINVAL;
    if (!all_finite(k, n) || !all_finite(l0, n)) return SS_EFALLBACK;
    *longest = 4;
    for (int32_t g = 0; g < n_labels; ++g) *longest = std::max(*longest, std::strlen(labels[g]));
    if (group)
        for (int64_t s = 0; s < n; ++s)
            if (group[s] >= n_labels) return SS_EINVAL;
    return SS_OK;
}

}  // namespace

extern "C" {

// sceneio.py:57-75 for the "masses" array: the text between "masses": [ and
// the closing bracket line (entries at indent 4, joined by ",\n").
int ss_doc_render_masses(int64_t n, const double *m, const double *x, const double *v, const double *f,
                         const uint8_t *fixed, char **out, int64_t *len) {
    if (!out || !len) return SS_EINVAL;
    const int rc = check_masses(n, m, x, v, f, fixed);
    if (rc) return rc;
    return render_blocks(n, kMassMax, mass_entry(m, x, v, f, fixed), out, len);
}

// The "springs" array; labels[g] is the JSON text of group g's label (the
// host escapes it), group[s] < 0 renders null.
int ss_doc_render_springs(int64_t n, const int64_t *si, const int64_t *sj, const double *k, const double *l0,
                          const int32_t *group, const char *const *labels, int32_t n_labels, char **out,
                          int64_t *len) {
    if (!out || !len) return SS_EINVAL;
    size_t longest = 0;
    const int rc = check_springs(n, si, sj, k, l0, group, labels, n_labels, &longest);
    if (rc) return rc;
    return render_blocks(n, kSpringFixed + longest, spring_entry(si, sj, k, l0, group, labels), out, len);
}

// The whole document: pre + masses entries + mid + springs entries + post
// (the host renders the small top-level values and passes the text around
// the two arrays), built in parallel into one buffer.
int ss_doc_render(int64_t n_masses, const double *m, const double *x, const double *v, const double *f,
                  const uint8_t *fixed, int64_t n_springs, const int64_t *si, const int64_t *sj, const double *k,
                  const double *l0, const int32_t *group, const char *const *labels, int32_t n_labels,
                  const char *pre, const char *mid, const char *post, char **out, int64_t *len) {
    if (!out || !len || !pre || !mid || !post) return SS_EINVAL;
    *out = nullptr;
    *len = 0;
    int rc = check_masses(n_masses, m, x, v, f, fixed);
    size_t longest = 0;
    if (rc || (rc = check_springs(n_springs, si, sj, k, l0, group, labels, n_labels, &longest))) return rc;
    const auto mp = render_parts(n_masses, kMassMax, mass_entry(m, x, v, f, fixed));
    const auto sp = render_parts(n_springs, kSpringFixed + longest, spring_entry(si, sj, k, l0, group, labels));
    const std::string a(pre), b(mid), c(post);
    std::vector<const std::string *> pieces{&a};
    for (const auto &q : mp) pieces.push_back(&q);
    pieces.push_back(&b);
    for (const auto &q : sp) pieces.push_back(&q);
    pieces.push_back(&c);
    return concat(pieces, out, len);
}

void ss_doc_free_text(char *p) { std::free(p); }

// Python repr of each of n doubles, '\n'-joined (tests).
int ss_doc_repr(int64_t n, const double *v, char **out, int64_t *len) {
    if (!out || !len || (n && !v)) return SS_EINVAL;
    if (!all_finite(v, n)) return SS_EINVAL;
    std::string s((size_t)n * 26, '\0');
    char *p = s.data();
    for (int64_t i = 0; i < n; ++i) {
        p = put_double(p, v[i]);
        *p++ = '\n';
    }
    s.resize((size_t)(p - s.data()));
    *out = static_cast<char *>(std::malloc(s.size() + 1));
    if (!*out) return SS_EINVAL;
    std::memcpy(*out, s.data(), s.size());
    *len = (int64_t)s.size();
    return SS_OK;
}

// Fast-path parse of an ASCII document (see the file header).
int ss_doc_parse(const char *text, int64_t len, ss_doc **out) {
    if (!text || len < 0 || !out) return SS_EINVAL;
    *out = nullptr;
    auto d = new ss_doc();
    Reader r{text, text + len};
    bool good = true;
    r.need('{');
    if (!r.ok || r.lit('}')) good = false;
    while (good) {
        const char *a;
        size_t n;
        if (!r.str(a, n)) {
            good = false;
            break;
        }
        std::string key(a, n);
        if (std::find(d->keys.begin(), d->keys.end(), key) != d->keys.end()) {
            good = false;                      // duplicate key: json.loads keeps the last, the slow path decides
            break;
        }
        r.need(':');
        r.ws();
        const int64_t start = (int64_t)(r.s - text);
        if (key == "masses") {
            good = read_array(r, [&](int64_t i) { return read_mass(r, *d, i); });
        } else if (key == "springs") {
            good = read_array(r, [&](int64_t i) { return read_spring(r, *d, i); });
        } else {
            r.skip();
            good = r.ok;
        }
        d->keys.push_back(key);
        d->off.push_back(start);
        d->span.push_back((int64_t)(r.s - text) - start);
        if (!good || !r.ok) {
            good = false;
            break;
        }
        if (r.lit(',')) continue;
        r.need('}');
        break;
    }
    r.ws();
    if (!good || !r.ok || r.s != r.e) {
        delete d;
        return SS_EFALLBACK;
    }
    const int64_t nm = (int64_t)d->m.size();
    for (size_t s = 0; s < d->si.size(); ++s)
        if (d->si[s] < 0 || d->si[s] >= nm || d->sj[s] < 0 || d->sj[s] >= nm) {
            delete d;                          // "no such mass": the slow path names the entry
            return SS_EFALLBACK;
        }
    *out = d;
    return SS_OK;
}

int ss_doc_info(const ss_doc *d, int64_t *n_masses, int64_t *n_springs, int32_t *n_keys, int32_t *n_labels) {
    if (!d) return SS_EINVAL;
    if (n_masses) *n_masses = (int64_t)d->m.size();
    if (n_springs) *n_springs = (int64_t)d->si.size();
    if (n_keys) *n_keys = (int32_t)d->keys.size();
    if (n_labels) *n_labels = (int32_t)d->labels.size();
    return SS_OK;
}

int ss_doc_key(const ss_doc *d, int32_t i, const char **name, int64_t *off, int64_t *len) {
    if (!d || i < 0 || i >= (int32_t)d->keys.size()) return SS_EINVAL;
    *name = d->keys[i].c_str();
    *off = d->off[i];
    *len = d->span[i];
    return SS_OK;
}

const char *ss_doc_label(const ss_doc *d, int32_t i) {
    return d && i >= 0 && i < (int32_t)d->labels.size() ? d->labels[i].c_str() : nullptr;
}

int ss_doc_masses(const ss_doc *d, double *m, double *x, double *v, double *f, uint8_t *fixed) {
    if (!d) return SS_EINVAL;
    const size_t n = d->m.size();
    if (n) {
        std::memcpy(m, d->m.data(), n * 8);
        std::memcpy(x, d->x.data(), n * 24);
        std::memcpy(v, d->v.data(), n * 24);
        std::memcpy(f, d->f.data(), n * 24);
        std::memcpy(fixed, d->fixed.data(), n);
    }
    return SS_OK;
}

int ss_doc_springs(const ss_doc *d, int64_t *si, int64_t *sj, double *k, double *l0, int32_t *group) {
    if (!d) return SS_EINVAL;
    const size_t n = d->si.size();
    if (n) {
        std::memcpy(si, d->si.data(), n * 8);
        std::memcpy(sj, d->sj.data(), n * 8);
        std::memcpy(k, d->k.data(), n * 8);
        std::memcpy(l0, d->l0.data(), n * 8);
        std::memcpy(group, d->group.data(), n * 4);
    }
    return SS_OK;
}

void ss_doc_free(ss_doc *d) { delete d; }

}  // extern "C"
