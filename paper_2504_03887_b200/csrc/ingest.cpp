// Native trace ingest and config digest.
//
// pm_ingest_json: chrome-trace JSON text -> the columns the reference's
// parse_trace builds (reference pkg/src/peakmem/trace.py:155-238): raw ts,
// dur, category, the seven integer args fields (INT64_MIN = None) and the
// names (interned: an id per event into a table of distinct names, UTF-8
// blob + code-point offsets), in FILE order, metadata records
// dropped, instants without a usable Addr/Bytes pair dropped.  It handles
// the common case exactly (numbers parsed with correctly rounded strtod,
// integers exact, floats truncated like int(), last duplicate key wins, JSON
// escapes decoded) and returns PM_INGEST_UNSUPPORTED for anything outside it
// (string-typed numbers, NaN / Infinity, non-object args, errors the
// reference reports with a message) so the caller's Python reader can take
// over with the reference's exact semantics.
//
// pm_bundle_digest: SHA-256 of json.dumps(payload, sort_keys=True,
// separators=(",", ":")) for the estimator's config digest
// (estimator.py:189-202; TraceBundle.to_json_dict, trace.py:116-143),
// streamed from the columns -- ensure_ascii escaping included.

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#if defined(__SSE2__)
#include <emmintrin.h>
#endif

#include <openssl/evp.h>

#include "../../include/peakmem_ingest.h"

namespace {

constexpr int64_t kNone = INT64_MIN;
enum { PM_INGEST_OK = 0 };
enum Cat { C_PF = 0, C_OP = 1, C_UA = 2, C_IN = 3, C_OTHER = 4 };
enum Field { F_PID = 0, F_PAR, F_SEQ, F_ADDR, F_BYTES, F_TA, F_TR, F_N };

thread_local std::string g_err;

struct Cols {
  std::vector<double> ts, dur;
  std::vector<int8_t> cat;
  std::vector<int64_t> ints[F_N];
  std::vector<int32_t> name_id;    // per event, into the table below
  // open-addressing set of the distinct names: slot -> name id + 1 (0 =
  // empty), keyed by the name's bytes in `names`; hash beside it
  std::vector<int32_t> slot;
  std::vector<uint64_t> slot_hash;
  int32_t n_names = 0;
  std::string names;               // distinct names, UTF-8
  std::vector<int64_t> name_off;   // code-point offsets, n_names+1
  std::vector<int64_t> name_boff;  // byte offsets into `names`, n_names+1
  int64_t dropped = 0;
  int64_t cp_total = 0;
  // rows parsed by the chunk threads, kept as they are (copied out in
  // parallel by pm_ingest_columns) with their name ids mapped into this
  // table: part k's rows follow this object's own rows and part k-1's
  std::vector<Cols> parts;
  std::vector<std::vector<int32_t>> remap;
  Cols() {
    name_off.push_back(0);
    name_boff.push_back(0);
  }
  int64_t rows() const {
    int64_t n = (int64_t)ts.size();
    for (const Cols& p : parts) n += (int64_t)p.ts.size();
    return n;
  }
};

// ---- JSON scanning -----------------------------------------------------------

struct Unsupported {};

struct Parser {
  const char* p;
  const char* end;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  // first byte at or after q that is '"', '\\' or a control character
  // (< 0x20), or end: 16 bytes per step where the buffer allows
  const char* run_end(const char* q) const {
#if defined(__SSE2__)
    const __m128i quote = _mm_set1_epi8('"'), bslash = _mm_set1_epi8('\\'),
                  ctl = _mm_set1_epi8(0x1F);
    while (end - q >= 16) {
      const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
      const __m128i hit = _mm_or_si128(
          _mm_or_si128(_mm_cmpeq_epi8(x, quote), _mm_cmpeq_epi8(x, bslash)),
          _mm_cmpeq_epi8(_mm_max_epu8(x, ctl), ctl));
      const int m = _mm_movemask_epi8(hit);
      if (m) return q + __builtin_ctz((unsigned)m);
      q += 16;
    }
#endif
    while (q < end && *q != '"' && *q != '\\' && (unsigned char)*q >= 0x20) ++q;
    return q;
  }
  // skip a string (p at its opening quote) with the same checks as str():
  // control characters, escapes and surrogate pairs
  void skip_str() {
    ++p;
    while (true) {
      p = run_end(p);
      if (p >= end) throw Unsupported();
      const char c = *p;
      if (c == '"') {
        ++p;
        return;
      }
      if (c != '\\') throw Unsupported();  // control character
      ++p;
      if (p >= end) throw Unsupported();
      const char e = *p++;
      switch (e) {
        case '"': case '\\': case '/': case 'b': case 'f': case 'n': case 'r':
        case 't':
          break;
        case 'u': {
          const uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (end - p < 6 || p[0] != '\\' || p[1] != 'u') throw Unsupported();
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) throw Unsupported();
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            throw Unsupported();
          }
          break;
        }
        default: throw Unsupported();
      }
    }
  }
  char peek() {
    ws();
    if (p >= end) throw Unsupported();
    return *p;
  }
  void expect(char c) {
    if (peek() != c) throw Unsupported();
    ++p;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out += (char)cp;
    } else if (cp < 0x800) {
      out += (char)(0xC0 | (cp >> 6));
      out += (char)(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += (char)(0xE0 | (cp >> 12));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    } else {
      out += (char)(0xF0 | (cp >> 18));
      out += (char)(0x80 | ((cp >> 12) & 0x3F));
      out += (char)(0x80 | ((cp >> 6) & 0x3F));
      out += (char)(0x80 | (cp & 0x3F));
    }
  }
  uint32_t hex4() {
    if (end - p < 4) throw Unsupported();
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else throw Unsupported();
    }
    return v;
  }
  // string -> UTF-8 (lone surrogates unsupported)
  std::string str() {
    expect('"');
    std::string out;
    const char* run = p;
    while (true) {
      p = run_end(p);
      if (p >= end) throw Unsupported();
      const unsigned char c = (unsigned char)*p;
      if (c == '"') {
        out.append(run, p - run);
        ++p;
        return out;
      }
      if (c < 0x20) throw Unsupported();
      out.append(run, p - run);
      ++p;
      if (p >= end) throw Unsupported();
      const char e = *p++;
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (end - p < 6 || p[0] != '\\' || p[1] != 'u') throw Unsupported();
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) throw Unsupported();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            throw Unsupported();
          }
          put_utf8(out, cp);
          break;
        }
        default: throw Unsupported();
      }
      run = p;
    }
  }
  // object key without copying when it has no escapes; escaped keys decode
  // into `scratch`
  std::string_view key(std::string& scratch) {
    expect('"');
    const char* s = p;
    p = run_end(p);
    if (p < end && *p == '"') {
      ++p;
      return {s, (size_t)(p - 1 - s)};
    }
    p = s - 1;
    scratch = str();
    return scratch;
  }
  // number token: kind 1 = integer, 2 = float
  int number(const char** s, const char** e) {
    ws();
    *s = p;
    if (p < end && *p == '-') ++p;
    if (p >= end || !(*p >= '0' && *p <= '9')) throw Unsupported();
    if (*p == '0' && p + 1 < end && p[1] >= '0' && p[1] <= '9')
      throw Unsupported();  // leading zero: invalid JSON
    int kind = 1;
    while (p < end && *p >= '0' && *p <= '9') ++p;
    if (p < end && *p == '.') {
      kind = 2;
      ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) throw Unsupported();
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      kind = 2;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) throw Unsupported();
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    *e = p;
    return kind;
  }
  void literal(const char* w) {
    const size_t n = strlen(w);
    if ((size_t)(end - p) < n || memcmp(p, w, n) != 0) throw Unsupported();
    p += n;
  }
  void skip() {
    const char c = peek();
    if (c == '{') {
      ++p;
      if (peek() == '}') { ++p; return; }
      while (true) {
        if (peek() != '"') throw Unsupported();
        skip_str();
        expect(':');
        skip();
        const char d = peek();
        ++p;
        if (d == '}') return;
        if (d != ',') throw Unsupported();
      }
    } else if (c == '[') {
      ++p;
      if (peek() == ']') { ++p; return; }
      while (true) {
        skip();
        const char d = peek();
        ++p;
        if (d == ']') return;
        if (d != ',') throw Unsupported();
      }
    } else if (c == '"') {
      skip_str();
    } else if (c == 't') {
      literal("true");
    } else if (c == 'f') {
      literal("false");
    } else if (c == 'n') {
      literal("null");
    } else {
      const char *s, *e;
      number(&s, &e);
    }
  }
};

// A scalar JSON value as the reference sees it after json.loads.
// Strings are views into the text unless they hold escapes (then decoded
// into `own`); a Val is filled in place and not copied.
struct Val {
  enum T { ABSENT, NUL, INT, FLT, STR, TRUE_, FALSE_, OTHER } t = ABSENT;
  int64_t i = 0;
  double f = 0;
  std::string_view s;
  std::string own;
};

void scalar(Parser& P, Val& v) {
  const char c = P.peek();
  if (c == '"') {
    v.t = Val::STR;
    v.s = P.key(v.own);
  } else if (c == 'n') {
    P.literal("null");
    v.t = Val::NUL;
  } else if (c == 't') {
    P.literal("true");
    v.t = Val::TRUE_;
  } else if (c == 'f') {
    P.literal("false");
    v.t = Val::FALSE_;
  } else if (c == '{' || c == '[') {
    P.skip();
    v.t = Val::OTHER;
  } else {
    const char *s, *e;
    const int kind = P.number(&s, &e);
    if (kind == 1) {
      const bool neg = *s == '-';
      uint64_t mag = 0;
      for (const char* q = s + neg; q < e; ++q) {
        if (__builtin_mul_overflow(mag, (uint64_t)10, &mag) ||
            __builtin_add_overflow(mag, (uint64_t)(*q - '0'), &mag))
          throw Unsupported();  // Python int beyond int64
      }
      if (mag > (neg ? (uint64_t)1 << 63 : (uint64_t)INT64_MAX)) throw Unsupported();
      v.t = Val::INT;
      v.i = neg ? (int64_t)(0 - mag) : (int64_t)mag;
      v.f = (double)v.i;  // float(int): round to nearest even
    } else {
      v.t = Val::FLT;
      // correctly rounded like Python's float(); overflow / underflow ->
      // out_of_range -> the Python reader decides
      const auto r = std::from_chars(s, e, v.f);
      if (r.ec != std::errc() || r.ptr != e || !std::isfinite(v.f))
        throw Unsupported();
    }
  }
}

// _as_int (trace.py:140-146): None -> None, int(value) otherwise
int64_t as_int(const Val& v) {
  switch (v.t) {
    case Val::ABSENT:
    case Val::NUL: return kNone;
    case Val::INT:
      if (v.i == kNone) throw Unsupported();
      return v.i;
    case Val::TRUE_: return 1;
    case Val::FALSE_: return 0;
    case Val::FLT: {
      const double t = std::trunc(v.f);
      if (!(t > -9.2e18 && t < 9.2e18)) throw Unsupported();
      return (int64_t)t;
    }
    default: throw Unsupported();  // strings / containers: Python path
  }
}

bool truthy(const Val& v) {  // `x or 0`
  switch (v.t) {
    case Val::INT: return v.i != 0;
    case Val::FLT: return v.f != 0.0;
    case Val::STR: return !v.s.empty();
    case Val::TRUE_: return true;
    default: return false;
  }
}

int32_t intern_name(Cols& C, std::string_view s) {
  const uint64_t h = std::hash<std::string_view>{}(s);
  if (2 * ((size_t)C.n_names + 1) > C.slot.size()) {
    // grow: re-place every name by its stored hash
    const size_t cap = std::max<size_t>(64, 2 * C.slot.size());
    std::vector<int32_t> slot(cap, 0);
    std::vector<uint64_t> sh(cap, 0);
    for (size_t k = 0; k < C.slot.size(); ++k) {
      if (C.slot[k] == 0) continue;
      size_t q = C.slot_hash[k] & (cap - 1);
      while (slot[q] != 0) q = (q + 1) & (cap - 1);
      slot[q] = C.slot[k];
      sh[q] = C.slot_hash[k];
    }
    C.slot.swap(slot);
    C.slot_hash.swap(sh);
  }
  const size_t mask = C.slot.size() - 1;
  size_t k = h & mask;
  for (; C.slot[k] != 0; k = (k + 1) & mask) {
    if (C.slot_hash[k] != h) continue;
    const int32_t id = C.slot[k] - 1;
    const int64_t b = C.name_boff[id], e = C.name_boff[id + 1];
    if ((size_t)(e - b) == s.size() && memcmp(C.names.data() + b, s.data(), s.size()) == 0)
      return id;
  }
  const int32_t id = C.n_names++;
  C.slot[k] = id + 1;
  C.slot_hash[k] = h;
  int64_t n = 0;
  for (unsigned char c : s)
    if ((c & 0xC0) != 0x80) ++n;
  C.cp_total += n;
  C.names.append(s.data(), s.size());
  C.name_off.push_back(C.cp_total);
  C.name_boff.push_back((int64_t)C.names.size());
  return id;
}

template <size_t N>
inline bool is(std::string_view k, const char (&w)[N]) {
  return k.size() == N - 1 && memcmp(k.data(), w, N - 1) == 0;
}

// one record object; appends a row or drops it
void record(Parser& P, Cols& C, bool strict) {
  if (P.peek() != '{') throw Unsupported();  // non-object record: error path
  ++P.p;
  std::string scratch;
  Val ph, cat, name, ts, dur;
  bool has_args = false;
  Val a[F_N];
  bool args_other = false;
  if (P.peek() == '}') {
    ++P.p;
  } else {
    while (true) {
      const auto key = P.key(scratch);
      P.expect(':');
      if (is(key, "ph")) scalar(P, ph);
      else if (is(key, "cat")) scalar(P, cat);
      else if (is(key, "name")) scalar(P, name);
      else if (is(key, "ts")) scalar(P, ts);
      else if (is(key, "dur")) scalar(P, dur);
      else if (is(key, "args")) {
        for (auto& x : a) x.t = Val::ABSENT;
        args_other = false;
        has_args = true;
        if (P.peek() == '{') {
          ++P.p;
          if (P.peek() == '}') {
            ++P.p;
          } else {
            while (true) {
              const auto k = P.key(scratch);
              P.expect(':');
              int f = -1;
              if (is(k, "Python id")) f = F_PID;
              else if (is(k, "Python parent id")) f = F_PAR;
              else if (is(k, "Sequence number")) f = F_SEQ;
              else if (is(k, "Addr")) f = F_ADDR;
              else if (is(k, "Bytes")) f = F_BYTES;
              else if (is(k, "Total Allocated")) f = F_TA;
              else if (is(k, "Total Reserved")) f = F_TR;
              if (f >= 0) scalar(P, a[f]);
              else P.skip();
              const char d = P.peek();
              ++P.p;
              if (d == '}') break;
              if (d != ',') throw Unsupported();
            }
          }
        } else {
          Val v;  // `args or {}`: falsy -> {}
          scalar(P, v);
          if (truthy(v) || v.t == Val::OTHER) args_other = true;
        }
      } else {
        P.skip();
      }
      const char d = P.peek();
      ++P.p;
      if (d == '}') break;
      if (d != ',') throw Unsupported();
    }
  }
  (void)has_args;
  if (ph.t == Val::STR && ph.s == "M") return;  // metadata record
  int category = C_OTHER;
  if (cat.t == Val::OTHER) throw Unsupported();  // unhashable: TypeError
  if (cat.t == Val::STR) {
    if (cat.s == "python_function") category = C_PF;
    else if (cat.s == "cpu_op") category = C_OP;
    else if (cat.s == "user_annotation") category = C_UA;
    else if (cat.s == "cpu_instant_event") category = C_IN;
    else if (cat.s != "other" && strict) throw Unsupported();
  } else if (strict) {
    throw Unsupported();
  }
  std::string_view nm;
  if (name.t == Val::STR) nm = name.s;
  else if (name.t != Val::ABSENT) throw Unsupported();  // str(non-string)
  if (ts.t != Val::INT && ts.t != Val::FLT) throw Unsupported();  // incl. missing
  double d = 0.0;
  if (dur.t == Val::INT || dur.t == Val::FLT) d = dur.f;
  else if (dur.t == Val::STR || dur.t == Val::OTHER) throw Unsupported();
  else if (dur.t == Val::TRUE_) d = 1.0;
  if (args_other && category != C_OTHER) throw Unsupported();
  int64_t out[F_N];
  for (int f = 0; f < F_N; ++f) out[f] = kNone;
  if (category == C_PF) {
    out[F_PID] = as_int(a[F_PID]);
    out[F_PAR] = as_int(a[F_PAR]);
  } else if (category == C_OP) {
    const int64_t s = as_int(a[F_SEQ]);
    out[F_SEQ] = (s != kNone && s < 0) ? kNone : s;
  } else if (category == C_IN) {
    const int64_t ad = as_int(a[F_ADDR]), nb = as_int(a[F_BYTES]);
    if (ad == kNone || nb == kNone || nb == 0) {
      if (strict) throw Unsupported();
      C.dropped += 1;
      return;
    }
    out[F_ADDR] = ad;
    out[F_BYTES] = nb;
    out[F_TA] = as_int(a[F_TA]);
    out[F_TR] = as_int(a[F_TR]);
  }
  C.ts.push_back(ts.f);
  C.dur.push_back(d);
  C.cat.push_back((int8_t)category);
  for (int f = 0; f < F_N; ++f) C.ints[f].push_back(out[f]);
  C.name_id.push_back(intern_name(C, nm));
}

// ---- SHA-256 --------------------------------------------------------------------

// OpenSSL's EVP SHA-256 (SHA-NI where the CPU has it, as Python's hashlib)
struct Sha256 {
  EVP_MD_CTX* ctx;
  Sha256() : ctx(EVP_MD_CTX_new()) { EVP_DigestInit_ex(ctx, EVP_sha256(), nullptr); }
  ~Sha256() { EVP_MD_CTX_free(ctx); }
  void update(const void* p, size_t n) { EVP_DigestUpdate(ctx, p, n); }
  void hex(char* out) {
    unsigned char d[32];
    unsigned int len = 0;
    EVP_DigestFinal_ex(ctx, d, &len);
    static const char* hx = "0123456789abcdef";
    for (int i = 0; i < 32; ++i) {
      out[2 * i] = hx[d[i] >> 4];
      out[2 * i + 1] = hx[d[i] & 15];
    }
    out[64] = 0;
  }
};

// streaming writer: buffered into the hash
// json.dumps string with ensure_ascii=True (py_encode_basestring_ascii)
void escape_json(std::string& b, const char* p, size_t n) {
  b += '"';
  size_t i = 0;
  while (i < n) {
    unsigned char c = (unsigned char)p[i];
    uint32_t cp;
    int len;
    if (c < 0x80) { cp = c; len = 1; }
    else if ((c >> 5) == 6) { cp = c & 0x1F; len = 2; }
    else if ((c >> 4) == 14) { cp = c & 0x0F; len = 3; }
    else { cp = c & 0x07; len = 4; }
    for (int k = 1; k < len && i + k < n; ++k) cp = (cp << 6) | (p[i + k] & 0x3F);
    i += len;
    switch (cp) {
      case '"': b += "\\\""; continue;
      case '\\': b += "\\\\"; continue;
      case '\n': b += "\\n"; continue;
      case '\r': b += "\\r"; continue;
      case '\t': b += "\\t"; continue;
      case '\b': b += "\\b"; continue;
      case '\f': b += "\\f"; continue;
      default: break;
    }
    if (cp >= 0x20 && cp <= 0x7E) {
      b += (char)cp;
    } else if (cp < 0x10000) {
      char t[8];
      snprintf(t, sizeof t, "\\u%04x", cp);
      b += t;
    } else {
      const uint32_t v = cp - 0x10000;
      char t[16];
      snprintf(t, sizeof t, "\\u%04x\\u%04x", 0xD800 | (v >> 10), 0xDC00 | (v & 0x3FF));
      b += t;
    }
  }
  b += '"';
}

struct Out {
  Sha256 sh;
  std::string b;
  void s(const char* x) { b += x; flush_maybe(); }
  void s(const std::string& x) { b += x; flush_maybe(); }
  void c(char x) { b += x; }
  void i(int64_t v) {
    char t[24];
    const auto r = std::to_chars(t, t + sizeof t, v);
    b.append(t, r.ptr - t);
  }
  void flush_maybe() {
    if (b.size() > (1u << 16)) flush_all();
  }
  void flush_all() {
    sh.update(b.data(), b.size());
    b.clear();
  }
  void str(const char* p, size_t n) {
    escape_json(b, p, n);
    flush_maybe();
  }
  void ilist(const int64_t* v, int64_t n) {
    c('[');
    for (int64_t k = 0; k < n; ++k) {
      if (k) c(',');
      i(v[k]);
    }
    c(']');
  }
  void done(char* hexout) {
    sh.update(b.data(), b.size());
    b.clear();
    sh.hex(hexout);
  }
};

// Strict UTF-8 validation (the reference reads the file with
// encoding="utf-8"; invalid input goes to the Python reader, which raises the
// reference's error).  ASCII runs are skipped 32 bytes at a time (SSE2) or 8.
bool valid_utf8(const unsigned char* p, const unsigned char* end) {
  while (p < end) {
#if defined(__SSE2__)
    // ASCII runs 32 bytes at a time
    while (end - p >= 32) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16));
      if (_mm_movemask_epi8(_mm_or_si128(a, b)) != 0) break;
      p += 32;
    }
#endif
    if (end - p >= 8) {
      uint64_t w;
      memcpy(&w, p, 8);
      if ((w & 0x8080808080808080ull) == 0) {
        p += 8;
        continue;
      }
    }
    const unsigned c = *p;
    if (c < 0x80) {
      ++p;
      continue;
    }
    int n;
    uint32_t cp;
    if ((c & 0xE0) == 0xC0) { n = 1; cp = c & 0x1F; }
    else if ((c & 0xF0) == 0xE0) { n = 2; cp = c & 0x0F; }
    else if ((c & 0xF8) == 0xF0) { n = 3; cp = c & 0x07; }
    else return false;
    if (end - p <= n) return false;
    for (int k = 1; k <= n; ++k) {
      if ((p[k] & 0xC0) != 0x80) return false;
      cp = (cp << 6) | (p[k] & 0x3F);
    }
    if ((n == 1 && cp < 0x80) || (n == 2 && cp < 0x800) || (n == 3 && cp < 0x10000) ||
        cp > 0x10FFFF || (cp >= 0xD800 && cp <= 0xDFFF))
      return false;
    p += n + 1;
  }
  return true;
}

// Adopt B as A's next part: B's distinct names are interned into A's table
// in B's first-occurrence order (so A's table is the one a sequential parse
// of A's text followed by B's would build); B's rows stay where they are.
void adopt_part(Cols& A, Cols&& B) {
  const size_t nb = B.name_boff.size() - 1;
  std::vector<int32_t> map(nb);
  for (size_t k = 0; k < nb; ++k)
    map[k] = intern_name(A, std::string_view(B.names).substr(
                                (size_t)B.name_boff[k],
                                (size_t)(B.name_boff[k + 1] - B.name_boff[k])));
  A.dropped += B.dropped;
  A.parts.push_back(std::move(B));
  A.remap.push_back(std::move(map));
}

// Parallel strict UTF-8 check: the text is cut at T points moved forward
// to a byte that starts a sequence (UTF-8 resynchronises there).
// parses running at once in this process: a parse's threads share the cores
// with the others (a thread pool of parse_trace calls would otherwise start
// cores x pool threads)
std::atomic<int> g_active_parses{0};

unsigned share_of_cores() {
  unsigned T = std::thread::hardware_concurrency();
  const char* env = getenv("PM_INGEST_SHARE");  // experiment: 0 = every parse uses all cores
  const int active = g_active_parses.load();
  if (!(env && atoi(env) == 0) && active > 1) T = std::max(1u, T / (unsigned)active);
  return T;
}

bool valid_utf8_parallel(const unsigned char* p, const unsigned char* end) {
  const size_t len = (size_t)(end - p);
  unsigned T = share_of_cores();
  if (T > 16) T = 16;
  if (len / T < (4u << 20)) T = (unsigned)(len >> 22);
  if (T < 2) return valid_utf8(p, end);
  std::vector<const unsigned char*> cut{p};
  for (unsigned t = 1; t < T; ++t) {
    const unsigned char* q = p + len * t / T;
    while (q < end && (*q & 0xC0) == 0x80) ++q;
    cut.push_back(q);
  }
  cut.push_back(end);
  std::vector<char> ok(T, 0);
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t)
    th.emplace_back([&, t] { ok[t] = valid_utf8(cut[t], cut[t + 1]); });
  ok[0] = valid_utf8(cut[0], cut[1]);
  for (auto& x : th) x.join();
  for (char o : ok)
    if (!o) return false;
  return true;
}

// The records of a JSON array, P.p just past its '['.  Large arrays are cut
// into chunks that start at "\n  {" (how profilers lay records out), parsed
// by one thread each; chunk t must stop exactly where chunk t+1 starts and
// the last must reach the ']' -- otherwise (a cut inside a record, an
// unsupported construct) the sequential loop below reparses the array, so
// the result is the sequential parse's either way.
void parse_records(Parser& P, Cols& C, bool strict) {
  const char* begin = P.p;
  const size_t len = (size_t)(P.end - begin);
  unsigned T = share_of_cores();
  if (T > 16) T = 16;
  if (len / T < (1u << 20)) T = (unsigned)(len >> 20);
  // records are laid out like the first one: a newline, its indentation,
  // '{' (profilers: "\n  {"); a first record not on its own line gives no
  // cut points
  std::string pat;
  const char* first = begin;
  while (first < P.end && (*first == ' ' || *first == '\n' || *first == '\r' ||
                           *first == '\t'))
    ++first;
  if (T >= 2 && first < P.end && *first == '{') {
    const char* nl = first;
    while (nl > begin && nl[-1] != '\n') --nl;
    if (nl > begin) pat = "\n" + std::string(nl, first) + "{";
  }
  std::vector<const char*> start{first};
  if (!pat.empty()) {
    for (unsigned t = 1; t < T; ++t) {
      const char* b = begin + len * t / T;
      const char* q = static_cast<const char*>(
          memmem(b, (size_t)(P.end - b), pat.data(), pat.size()));
      if (q && q + pat.size() - 1 > start.back()) start.push_back(q + pat.size() - 1);
    }
  }
  if (start.size() >= 2) {
    const size_t nt = start.size();
    std::vector<Cols> part(nt);
    std::vector<const char*> stop(nt, nullptr);
    std::vector<char> closed(nt, 0), ok(nt, 0);
    auto work = [&](size_t t) {
      try {
        Parser Q{start[t], P.end};
        const char* next = t + 1 < nt ? start[t + 1] : nullptr;
        if (Q.peek() == ']') {  // empty array
          ++Q.p;
          closed[t] = 1;
          stop[t] = Q.p;
          ok[t] = 1;
          return;
        }
        while (true) {
          record(Q, part[t], strict);
          const char d = Q.peek();
          ++Q.p;
          if (d == ']') {
            closed[t] = 1;
            break;
          }
          if (d != ',') return;
          Q.ws();
          if (next && Q.p >= next) break;
        }
        stop[t] = Q.p;
        ok[t] = 1;
      } catch (...) {
      }
    };
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    bool good = true;
    for (size_t t = 0; t < nt && good; ++t) {
      good = ok[t] && (t + 1 < nt ? (!closed[t] && stop[t] == start[t + 1]) : closed[t]);
    }
    if (good) {
      for (size_t t = 0; t < nt; ++t) adopt_part(C, std::move(part[t]));
      P.p = stop[nt - 1];
      return;
    }
  }
  // sequential
  if (P.peek() == ']') {
    ++P.p;
    return;
  }
  while (true) {
    record(P, C, strict);
    const char d = P.peek();
    ++P.p;
    if (d == ']') break;
    if (d != ',') throw Unsupported();
  }
}

}  // namespace

extern "C" {

const char* pm_ingest_last_error(void) { return g_err.c_str(); }

// Parse; *handle receives an opaque column set (pm_ingest_free).  Returns 0,
// PM_INGEST_UNSUPPORTED (5: use the Python reader) or PM_INGEST_EMPTY (7).
int pm_ingest_json(const char* text, int64_t len, int strict, void** handle) {
  *handle = nullptr;
  g_active_parses.fetch_add(1);
  struct Leave {
    ~Leave() { g_active_parses.fetch_sub(1); }
  } leave;
  if (!valid_utf8_parallel(reinterpret_cast<const unsigned char*>(text),
                           reinterpret_cast<const unsigned char*>(text) + len)) {
    g_err = "input is not valid UTF-8";
    return PM_INGEST_UNSUPPORTED;
  }
  Cols* C = new Cols();
  Parser P{text, text + len};
  try {
    const char c = P.peek();
    if (c == '{') {
      ++P.p;
      bool found = false;
      if (P.peek() != '}') {
        while (true) {
          const std::string key = P.str();
          P.expect(':');
          if (key == "traceEvents") {
            if (found) throw Unsupported();  // duplicate key: last wins, rare
            found = true;
            P.expect('[');
            parse_records(P, *C, strict != 0);
          } else {
            P.skip();
          }
          const char d = P.peek();
          ++P.p;
          if (d == '}') break;
          if (d != ',') throw Unsupported();
        }
      } else {
        ++P.p;
      }
      if (!found) throw Unsupported();
    } else if (c == '[') {
      ++P.p;
      parse_records(P, *C, strict != 0);
    } else {
      throw Unsupported();
    }
    P.ws();
    if (P.p != P.end) throw Unsupported();
  } catch (const Unsupported&) {
    delete C;
    g_err = "outside the native reader's subset";
    return PM_INGEST_UNSUPPORTED;
  }
  if (C->rows() == 0) {
    delete C;
    return PM_INGEST_EMPTY;
  }
  *handle = C;
  return PM_INGEST_OK;
}

int64_t pm_ingest_count(void* h) { return static_cast<Cols*>(h)->rows(); }
int64_t pm_ingest_dropped(void* h) { return static_cast<Cols*>(h)->dropped; }
int64_t pm_ingest_n_names(void* h) { return static_cast<Cols*>(h)->n_names; }
int64_t pm_ingest_names_bytes(void* h) { return (int64_t)static_cast<Cols*>(h)->names.size(); }

// Copy the columns out: ints is F_N x n (field-major: python id, parent id,
// sequence number, addr, bytes, total allocated, total reserved); name_id
// (n) indexes the distinct-name table (name_off: n_names+1 code points).
void pm_ingest_columns(void* h, double* ts, double* dur, int8_t* cat,
                       int64_t* ints, int32_t* name_id, int64_t* name_off,
                       char* names) {
  Cols* C = static_cast<Cols*>(h);
  const size_t n = (size_t)C->rows();
  // one copy job per row block (this object's own rows, then each part),
  // run in parallel; part name ids are mapped into the merged table
  auto copy_block = [&](const Cols& B, size_t at, const std::vector<int32_t>* map) {
    const size_t m = B.ts.size();
    memcpy(ts + at, B.ts.data(), m * sizeof(double));
    memcpy(dur + at, B.dur.data(), m * sizeof(double));
    memcpy(cat + at, B.cat.data(), m);
    for (int f = 0; f < F_N; ++f)
      memcpy(ints + f * n + at, B.ints[f].data(), m * sizeof(int64_t));
    if (map) {
      for (size_t i = 0; i < m; ++i) name_id[at + i] = (*map)[B.name_id[i]];
    } else {
      memcpy(name_id + at, B.name_id.data(), m * sizeof(int32_t));
    }
  };
  std::vector<std::thread> th;
  size_t at = C->ts.size();
  for (size_t k = 0; k < C->parts.size(); ++k) {
    th.emplace_back(copy_block, std::cref(C->parts[k]), at, &C->remap[k]);
    at += C->parts[k].ts.size();
  }
  copy_block(*C, 0, nullptr);
  for (auto& x : th) x.join();
  memcpy(name_off, C->name_off.data(), C->name_off.size() * sizeof(int64_t));
  memcpy(names, C->names.data(), C->names.size());
}

void pm_ingest_free(void* h) { delete static_cast<Cols*>(h); }

// SHA-256 of the estimator payload (estimator.py:189-202) from columns in
// event-id order.  name_id (n) indexes a table of n_names names: UTF-8
// blob + BYTE offsets (n_names+1).  ints as in
// pm_ingest_columns.  sidecar_present 0 -> "sidecar": null.  max_split < 0
// -> null.  Writes 64 hex chars + NUL to hex_out.
int pm_bundle_digest(int64_t n, const int8_t* cat, const int64_t* start,
                     const int64_t* dur, const int64_t* ints,
                     const int32_t* name_id, int64_t n_names,
                     const char* names, const int64_t* name_off,
                     int sidecar_present, const int64_t* param_sizes,
                     int64_t n_param, const int64_t* batch_bytes,
                     int64_t n_batch, const char* optimizer,
                     int64_t opt_len, int64_t sc_capacity, int64_t sc_initial,
                     int64_t iterations, int64_t device_capacity,
                     int64_t initial_memory, int64_t max_split,
                     char* hex_out) {
  static const char* cats[5] = {"python_function", "cpu_op", "user_annotation",
                                "cpu_instant_event", "other"};
  // args keys in sort order and their field index
  static const struct { const char* k; int f; } args[7] = {
      {"Addr", F_ADDR}, {"Bytes", F_BYTES}, {"Python id", F_PID},
      {"Python parent id", F_PAR}, {"Sequence number", F_SEQ},
      {"Total Allocated", F_TA}, {"Total Reserved", F_TR}};
  std::vector<std::string> esc((size_t)n_names);
  for (int64_t k = 0; k < n_names; ++k)
    escape_json(esc[k], names + name_off[k], (size_t)(name_off[k + 1] - name_off[k]));
  Out o;
  o.s("{\"device_capacity\":");
  o.i(device_capacity);
  o.s(",\"initial_memory\":");
  o.i(initial_memory);
  o.s(",\"iterations\":");
  o.i(iterations);
  o.s(",\"max_split_size\":");
  if (max_split < 0) o.s("null");
  else o.i(max_split);
  o.s(",\"sidecar\":");
  if (!sidecar_present) {
    o.s("null");
  } else {
    o.s("{\"batch_bytes\":");
    o.ilist(batch_bytes, n_batch);
    o.s(",\"device_capacity_bytes\":");
    o.i(sc_capacity);
    o.s(",\"initial_memory_bytes\":");
    o.i(sc_initial);
    o.s(",\"optimizer\":");
    o.str(optimizer, (size_t)opt_len);
    o.s(",\"param_sizes\":");
    o.ilist(param_sizes, n_param);
    o.c('}');
  }
  o.s(",\"trace\":{\"traceEvents\":[");
  o.flush_all();
  // the events: fixed-length pieces memcpy'd and digits written in place
  // into a raw buffer handed to the hash every ~64 KB (std::string appends
  // with strlen per piece cost ~10x more per event)
  {
    struct Piece { const char* p; size_t n; };
    Piece key[7], catp[5];
    for (int k = 0; k < 7; ++k) {
      static thread_local std::string kb[7];
      kb[k] = std::string("\"") + args[k].k + "\":";
      key[k] = {kb[k].data(), kb[k].size()};
    }
    for (int k = 0; k < 5; ++k) catp[k] = {cats[k], strlen(cats[k])};
    size_t max_name = 0;
    for (const std::string& x : esc) max_name = std::max(max_name, x.size());
    const size_t max_event = 512 + max_name;
    static const char kArgs[] = "{\"args\":{";
    static const char kCat[] = "},\"cat\":\"";
    static const char kDur[] = "\",\"dur\":";
    static const char kName[] = ",\"name\":";
    static const char kPhI[] = ",\"ph\":\"i\",\"ts\":";
    static const char kPhX[] = ",\"ph\":\"X\",\"ts\":";
    // one event at B + pos (room for max_event bytes guaranteed)
    auto emit = [&](char* B, size_t& pos, int64_t e) {
      auto put = [&](const char* p, size_t m) {
        memcpy(B + pos, p, m);
        pos += m;
      };
      auto num = [&](int64_t v) {
        pos = (size_t)(std::to_chars(B + pos, B + pos + 24, v).ptr - B);
      };
      if (e) B[pos++] = ',';
      put(kArgs, sizeof kArgs - 1);
      bool first = true;
      for (int k = 0; k < 7; ++k) {
        const int64_t v = ints[args[k].f * n + e];
        if (v == kNone) continue;
        if (!first) B[pos++] = ',';
        first = false;
        put(key[k].p, key[k].n);
        num(v);
      }
      put(kCat, sizeof kCat - 1);
      const Piece& cp = catp[cat[e] < 0 || cat[e] > 4 ? 4 : cat[e]];
      put(cp.p, cp.n);
      put(kDur, sizeof kDur - 1);
      num(dur[e]);
      put(kName, sizeof kName - 1);
      const std::string& nm = esc[name_id[e]];
      put(nm.data(), nm.size());
      if (cat[e] == C_IN)
        put(kPhI, sizeof kPhI - 1);
      else
        put(kPhX, sizeof kPhX - 1);
      num(start[e]);
      B[pos++] = '}';
    };
    const size_t cap = std::max<size_t>(1 << 18, 2 * max_event);
    if (n < 20000 || std::thread::hardware_concurrency() < 2) {
      std::vector<char> buf(cap);
      size_t pos = 0;
      for (int64_t e = 0; e < n; ++e) {
        if (pos + max_event > cap) {
          o.sh.update(buf.data(), pos);
          pos = 0;
        }
        emit(buf.data(), pos, e);
      }
      o.sh.update(buf.data(), pos);
    } else {
      // a formatter thread fills a ring of buffers while this thread hashes
      // them in order: formatting and SHA-256 overlap
      constexpr int K = 4;
      std::vector<std::vector<char>> ring(K, std::vector<char>(cap));
      std::atomic<int> ready[K];
      size_t len[K];
      for (int k = 0; k < K; ++k) ready[k].store(0);
      std::atomic<int64_t> sealed{-1};  // total buffers, once known
      std::thread fmt([&] {
        int64_t b = 0;
        size_t pos = 0;
        auto seal = [&] {
          const int slot = (int)(b % K);
          len[slot] = pos;
          ready[slot].store(1, std::memory_order_release);
          ++b;
          pos = 0;
          const int next = (int)(b % K);
          while (ready[next].load(std::memory_order_acquire) != 0)
            std::this_thread::yield();
        };
        for (int64_t e = 0; e < n; ++e) {
          if (pos + max_event > cap) seal();
          emit(ring[b % K].data(), pos, e);
        }
        seal();
        sealed.store(b, std::memory_order_release);
      });
      for (int64_t i = 0;; ++i) {
        const int slot = (int)(i % K);
        for (;;) {
          if (ready[slot].load(std::memory_order_acquire)) break;
          const int64_t t = sealed.load(std::memory_order_acquire);
          if (t >= 0 && i >= t) break;
          std::this_thread::yield();
        }
        const int64_t t = sealed.load(std::memory_order_acquire);
        if (!ready[slot].load(std::memory_order_acquire) && t >= 0 && i >= t) break;
        o.sh.update(ring[slot].data(), len[slot]);
        ready[slot].store(0, std::memory_order_release);
      }
      fmt.join();
    }
  }
  o.s("]}}");
  o.done(hex_out);
  return 0;
}

}  // extern "C"
