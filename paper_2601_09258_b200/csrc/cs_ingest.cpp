// cs_ingest.cpp — native Chrome-trace JSON ingest.
//
// Replaces the reference's parse_trace_json (trace_io.cpp:162-206, per record
// parse_record 87-158) followed by the interning every exporter does
// (names in lexicographic order, forward_mode class, batch/workload table,
// (name, commHash, rank) collective slots, counter values), producing the
// cs_event records the device consumes directly, without a DOM.
//
// Semantics follow the reference as built with nlohmann/json 3.11:
//  * the document must be valid JSON (RFC 8259 as nlohmann enforces it:
//    UTF-8 checked, no leading zeros, no control characters in strings, no
//    float overflowing to infinity); otherwise the trace is empty with one
//    issue (on an overflowing float the reference itself terminates);
//  * events: a top-level array, or the last "traceEvents" array member of a
//    top-level object;
//  * duplicate object keys: the last one wins; args are flattened in sorted
//    key order ("a.b" for objects, "a.0" for arrays), later writes win;
//  * numbers: integer syntax -> int64 / uint64 (else double), fraction or
//    exponent -> double (strtod, correctly rounded); ts/dur as double,
//    us -> ns by llround(us * 1000.0);
//  * ph "M" is dropped silently, unknown phases / categories are warnings,
//    type errors drop the record with an issue;
//  * fallback event ids are next_id = max(next_id, eid) + 1 over kept
//    records in document order; events are then stable-sorted by
//    (start_ts, event_id) (trace.hpp:110-113).
// The split into records is one sequential scan; records parse in parallel.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cerrno>
#include <cstring>
#include <deque>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <string_view>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <variant>
#include <vector>

#include <emmintrin.h>

#include "cs_parallel.h"
#include "cs_guard.h"
#include "cyclescope_b200.h"

struct cs_ingest_result {
  std::vector<cs_event> events;
  std::vector<uint64_t> event_ids;
  std::vector<cs_workload> workloads;
  std::string names_packed;
  uint32_t n_names = 0;
  std::vector<int32_t> comm_name, comm_rank;
  // resolve_topology (align.cpp:178-191): per comm slot a location, -1 unmapped
  std::vector<int32_t> comm_location, loc_device;
  std::string loc_nodes_packed;
  int topology_conflict = 0;
  std::vector<std::tuple<std::string, int, std::string, int>> topo;  // (hash, rank, node, device)
  // clock domains (src.clock, default "reference") and inline beacons
  // (extract_beacons, align.cpp:86-95): per event a domain id, the sorted
  // domain names, and (event index, reference_ts) in event order
  std::vector<uint16_t> domain;
  std::vector<std::string> domains;
  std::vector<std::pair<uint64_t, int64_t>> beacons;
  bool calibrated = false;
  std::string comm_hash_packed;
  uint64_t n_issues = 0;  // parse issues
  std::vector<cs_ingest_issue> issues;  // parse issues, then validate_trace's
  uint64_t categories[8] = {};
  uint64_t n_errors = 0;
  void issue(uint8_t sev, uint8_t code, bool has_id, uint64_t id) {
    cs_ingest_issue x{};
    x.severity = sev;
    x.code = code;
    x.has_event_id = has_id ? 1 : 0;
    x.event_id = has_id ? id : 0;
    issues.push_back(x);
    n_errors += sev == CS_SEV_ERROR;
  }
};

namespace {

struct BadJson {};  // a syntax error anywhere: the whole document is rejected
struct TypeError {};  // a json::exception inside one record: the record is dropped

// ------------------------------------------------------------ scanner
struct Scanner {
  const char* p;
  const char* end;

  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  char peek() {
    ws();
    if (p >= end) throw BadJson{};
    return *p;
  }
  void expect(char c) {
    if (peek() != c) throw BadJson{};
    ++p;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
    if (cp < 0x80) {
      out.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  uint32_t hex4() {
    if (end - p < 4) throw BadJson{};
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else throw BadJson{};
    }
    return v;
  }
  // one UTF-8 sequence starting at p (first byte >= 0x80), validated as
  // nlohmann's lexer does (shortest form, no surrogates, <= U+10FFFF)
  void utf8(std::string* out) {
    const auto b0 = static_cast<unsigned char>(*p);
    int n;
    unsigned char lo = 0x80, hi = 0xBF;
    if (b0 >= 0xC2 && b0 <= 0xDF) n = 1;
    else if (b0 == 0xE0) { n = 2; lo = 0xA0; }
    else if ((b0 >= 0xE1 && b0 <= 0xEC) || b0 == 0xEE || b0 == 0xEF) n = 2;
    else if (b0 == 0xED) { n = 2; hi = 0x9F; }
    else if (b0 == 0xF0) { n = 3; lo = 0x90; }
    else if (b0 >= 0xF1 && b0 <= 0xF3) n = 3;
    else if (b0 == 0xF4) { n = 3; hi = 0x8F; }
    else throw BadJson{};
    if (end - p < n + 1) throw BadJson{};
    for (int i = 1; i <= n; ++i) {
      const auto b = static_cast<unsigned char>(p[i]);
      if (b < (i == 1 ? lo : 0x80) || b > (i == 1 ? hi : 0xBF)) throw BadJson{};
    }
    if (out) out->append(p, n + 1);
    p += n + 1;
  }
  // string at p (opening quote), decoded into *out when given
  void string(std::string* out) {
    expect('"');
    while (true) {
      if (p >= end) throw BadJson{};
      const auto c = static_cast<unsigned char>(*p);
      if (c == '"') {
        ++p;
        return;
      }
      if (c < 0x20) throw BadJson{};
      if (c == '\\') {
        ++p;
        if (p >= end) throw BadJson{};
        const char e = *p++;
        char lit = 0;
        switch (e) {
          case '"': lit = '"'; break;
          case '\\': lit = '\\'; break;
          case '/': lit = '/'; break;
          case 'b': lit = '\b'; break;
          case 'f': lit = '\f'; break;
          case 'n': lit = '\n'; break;
          case 'r': lit = '\r'; break;
          case 't': lit = '\t'; break;
          case 'u': {
            uint32_t cp = hex4();
            if (cp >= 0xD800 && cp <= 0xDBFF) {
              if (end - p < 2 || p[0] != '\\' || p[1] != 'u') throw BadJson{};
              p += 2;
              const uint32_t lo = hex4();
              if (lo < 0xDC00 || lo > 0xDFFF) throw BadJson{};
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
            } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
              throw BadJson{};
            }
            if (out) put_utf8(*out, cp);
            continue;
          }
          default: throw BadJson{};
        }
        if (out) out->push_back(lit);
        continue;
      }
      if (c >= 0x80) {
        utf8(out);
        continue;
      }
      // run of plain ASCII
      const char* q = p;
      while (q < end && static_cast<unsigned char>(*q) >= 0x20 && *q != '"' && *q != '\\' &&
             static_cast<unsigned char>(*q) < 0x80)
        ++q;
      if (out) out->append(p, static_cast<size_t>(q - p));
      p = q;
    }
  }
  // string at p as a view into the document when it has no escapes (the
  // common case), else decoded into buf; validated either way
  std::string_view str_view(std::string& buf) {
    if (peek() != '"') throw BadJson{};
    const char* b = p + 1;
    const char* q = b;
    while (q < end && *q != '"' && *q != '\\' && static_cast<unsigned char>(*q) >= 0x20 &&
           static_cast<unsigned char>(*q) < 0x80)
      ++q;
    if (q < end && *q == '"') {
      p = q + 1;
      return std::string_view(b, static_cast<size_t>(q - b));
    }
    buf.clear();
    string(&buf);
    return std::string_view(buf);
  }
  // structural skip of a value (strings tracked, nothing else validated):
  // used to split the events array; every record is validated by its parser
  static const uint8_t* structural_table() {
    static const auto t = [] {
      static uint8_t x[256] = {};
      x[static_cast<uint8_t>('"')] = 1;
      x[static_cast<uint8_t>('{')] = 2;
      x[static_cast<uint8_t>('[')] = 2;
      x[static_cast<uint8_t>('}')] = 3;
      x[static_cast<uint8_t>(']')] = 3;
      return x;
    }();
    return t;
  }
  void skip_string_raw() {  // p just after the opening quote
    while (p < end) {
      const char c = *p++;
      if (c == '"') return;
      if (c == '\\') ++p;  // the escaped character, whatever it is
    }
    throw BadJson{};
  }
  // next byte at or after q that is one of " \\ { } [ ] (SSE2, 16 bytes a step)
  static const char* next_special(const char* q, const char* e) {
    const __m128i dq = _mm_set1_epi8('"'), bs = _mm_set1_epi8('\\');
    const __m128i lb = _mm_set1_epi8('{'), rb = _mm_set1_epi8('}');
    const __m128i ls = _mm_set1_epi8('['), rs = _mm_set1_epi8(']');
    while (e - q >= 16) {
      const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
      const __m128i m = _mm_or_si128(
          _mm_or_si128(_mm_or_si128(_mm_cmpeq_epi8(v, dq), _mm_cmpeq_epi8(v, bs)),
                       _mm_or_si128(_mm_cmpeq_epi8(v, lb), _mm_cmpeq_epi8(v, rb))),
          _mm_or_si128(_mm_cmpeq_epi8(v, ls), _mm_cmpeq_epi8(v, rs)));
      const int bits = _mm_movemask_epi8(m);
      if (bits) return q + __builtin_ctz(static_cast<unsigned>(bits));
      q += 16;
    }
    while (q < e && *q != '"' && *q != '\\' && *q != '{' && *q != '}' && *q != '[' && *q != ']') ++q;
    return q;
  }
  // next byte that is one of " \\ { } [ ] ,
  static const char* next_special_comma(const char* q, const char* e) {
    const __m128i dq = _mm_set1_epi8('"'), bs = _mm_set1_epi8('\\');
    const __m128i lb = _mm_set1_epi8('{'), rb = _mm_set1_epi8('}');
    const __m128i ls = _mm_set1_epi8('['), rs = _mm_set1_epi8(']'), cm = _mm_set1_epi8(',');
    while (e - q >= 16) {
      const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
      const __m128i m = _mm_or_si128(
          _mm_or_si128(_mm_or_si128(_mm_cmpeq_epi8(v, dq), _mm_cmpeq_epi8(v, bs)),
                       _mm_or_si128(_mm_cmpeq_epi8(v, lb), _mm_cmpeq_epi8(v, rb))),
          _mm_or_si128(_mm_or_si128(_mm_cmpeq_epi8(v, ls), _mm_cmpeq_epi8(v, rs)),
                       _mm_cmpeq_epi8(v, cm)));
      const int bits = _mm_movemask_epi8(m);
      if (bits) return q + __builtin_ctz(static_cast<unsigned>(bits));
      q += 16;
    }
    while (q < e && *q != '"' && *q != '\\' && *q != '{' && *q != '}' && *q != '[' &&
           *q != ']' && *q != ',')
      ++q;
    return q;
  }
  // next quote or backslash (inside a string)
  static const char* next_quote(const char* q, const char* e) {
    const __m128i dq = _mm_set1_epi8('"'), bs = _mm_set1_epi8('\\');
    while (e - q >= 16) {
      const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
      const int bits = _mm_movemask_epi8(_mm_or_si128(_mm_cmpeq_epi8(v, dq), _mm_cmpeq_epi8(v, bs)));
      if (bits) return q + __builtin_ctz(static_cast<unsigned>(bits));
      q += 16;
    }
    while (q < e && *q != '"' && *q != '\\') ++q;
    return q;
  }
  void skip_structural() {
    const char c = peek();
    if (c != '{' && c != '[' && c != '"') {
      while (p < end && *p != ',' && *p != ']' && *p != '}' && *p != ' ' && *p != '\n' &&
             *p != '\t' && *p != '\r')
        ++p;
      return;
    }
    int depth = 0;
    bool in_str = false;
    while (p < end) {
      p = in_str ? next_quote(p, end) : next_special(p, end);
      if (p >= end) break;
      const char x = *p++;
      if (x == '\\') {
        ++p;  // escaped character (only inside strings in valid JSON)
      } else if (x == '"') {
        in_str = !in_str;
        if (!in_str && depth == 0) return;  // a top-level string value
      } else if (x == '{' || x == '[') {
        ++depth;
      } else if (--depth == 0) {
        return;
      }
    }
    throw BadJson{};
  }
  // number syntax check; returns [begin, end) and whether integer syntax
  std::string_view number(bool* is_int) {
    ws();
    const char* b = p;
    if (p < end && *p == '-') ++p;
    if (p >= end) throw BadJson{};
    if (*p == '0') {
      ++p;
    } else if (*p >= '1' && *p <= '9') {
      while (p < end && *p >= '0' && *p <= '9') ++p;
    } else {
      throw BadJson{};
    }
    bool integer = true;
    if (p < end && *p == '.') {
      integer = false;
      ++p;
      if (p >= end || *p < '0' || *p > '9') throw BadJson{};
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      integer = false;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || *p < '0' || *p > '9') throw BadJson{};
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    *is_int = integer;
    // nlohmann rejects floats that overflow to +-inf (out_of_range 406; the
    // reference's parse_trace_json does not catch it and terminates): here the
    // whole document is rejected.  Only long mantissas or large exponents can
    // overflow, so strtod runs on those alone.
    if (!integer && (p - b > 300 || has_big_exponent(b, p))) {
      const std::string tok(b, p);
      if (!std::isfinite(std::strtod(tok.c_str(), nullptr))) throw BadJson{};
    }
    return std::string_view(b, static_cast<size_t>(p - b));
  }
  static bool has_big_exponent(const char* b, const char* e) {
    const char* x = b;
    while (x < e && *x != 'e' && *x != 'E') ++x;
    if (x == e) return false;
    ++x;
    if (x < e && (*x == '+' || *x == '-')) {
      if (*x == '-') return false;
      ++x;
    }
    return e - x >= 3;  // |exponent| >= 100
  }
  void literal(const char* lit) {
    const size_t n = std::strlen(lit);
    if (static_cast<size_t>(end - p) < n || std::memcmp(p, lit, n) != 0) throw BadJson{};
    p += n;
  }
  // any value, validated and skipped
  void skip() {
    const char c = peek();
    if (c == '"') {
      string(nullptr);
    } else if (c == '{') {
      ++p;
      if (peek() == '}') {
        ++p;
        return;
      }
      while (true) {
        string(nullptr);
        expect(':');
        skip();
        const char d = peek();
        ++p;
        if (d == '}') return;
        if (d != ',') throw BadJson{};
      }
    } else if (c == '[') {
      ++p;
      if (peek() == ']') {
        ++p;
        return;
      }
      while (true) {
        skip();
        const char d = peek();
        ++p;
        if (d == ']') return;
        if (d != ',') throw BadJson{};
      }
    } else if (c == 't') {
      literal("true");
    } else if (c == 'f') {
      literal("false");
    } else if (c == 'n') {
      literal("null");
    } else {
      bool i = false;
      number(&i);
    }
  }
};

// ------------------------------------------------------------ values
// A parsed JSON number as nlohmann classifies it.
struct Num {
  enum T { Int, Uint, Float } t;
  int64_t i = 0;
  uint64_t u = 0;
  double f = 0.0;
};

// Integers are converted by hand (overflow: nlohmann's float fallback via
// strtod); floats take Clinger's exact fast path when the decimal mantissa
// has <= 15 digits and |exponent| <= 22 (one correctly rounded IEEE operation
// on exact operands == strtod), strtod otherwise.
Num parse_number(std::string_view s, bool is_int) {
  Num n{Num::Float};
  const char* c = s.data();
  const char* e = c + s.size();
  const bool neg = *c == '-';
  const char* d = neg ? c + 1 : c;
  if (is_int) {
    if (e - d <= 18) {  // < 1e18: exact in int64 / uint64
      uint64_t v = 0;
      for (const char* q = d; q < e; ++q) v = v * 10 + static_cast<uint64_t>(*q - '0');
      if (neg) {
        n.t = Num::Int;
        n.i = -static_cast<int64_t>(v);
      } else {
        n.t = Num::Uint;
        n.u = v;
      }
      return n;
    }
    std::string tmp(s);
    errno = 0;
    if (neg) {
      const long long v = std::strtoll(tmp.c_str(), nullptr, 10);
      if (errno == 0) {
        n.t = Num::Int;
        n.i = v;
        return n;
      }
    } else {
      const unsigned long long v = std::strtoull(tmp.c_str(), nullptr, 10);
      if (errno == 0) {
        n.t = Num::Uint;
        n.u = v;
        return n;
      }
    }
    n.f = std::strtod(tmp.c_str(), nullptr);
    return n;
  }
  // mantissa digits and decimal exponent
  uint64_t m = 0;
  int digits = 0, exp10 = 0;
  const char* q = d;
  bool fast = true;
  for (; q < e && *q >= '0' && *q <= '9'; ++q) {
    if (m || *q != '0') {
      m = m * 10 + static_cast<uint64_t>(*q - '0');
      ++digits;
    }
  }
  if (q < e && *q == '.') {
    for (++q; q < e && *q >= '0' && *q <= '9'; ++q) {
      if (m || *q != '0') {
        m = m * 10 + static_cast<uint64_t>(*q - '0');
        ++digits;
      }
      --exp10;
    }
  }
  if (q < e && (*q == 'e' || *q == 'E')) {
    ++q;
    const bool eneg = *q == '-';
    if (*q == '+' || *q == '-') ++q;
    int x = 0;
    for (; q < e; ++q) {
      if (x > 10000) {
        fast = false;
        break;
      }
      x = x * 10 + (*q - '0');
    }
    exp10 += eneg ? -x : x;
  }
  static const double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                     1e8,  1e9,  1e10, 1e11, 1e12, 1e13, 1e14, 1e15,
                                     1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  if (fast && digits <= 15 && exp10 >= -22 && exp10 <= 22) {
    double v = static_cast<double>(m);
    v = exp10 < 0 ? v / kPow10[-exp10] : v * kPow10[exp10];
    n.f = neg ? -v : v;
    return n;
  }
  std::string tmp(s);
  n.f = std::strtod(tmp.c_str(), nullptr);
  return n;
}

double num_as_double(const Num& n) {  // get<double>() on a number
  switch (n.t) {
    case Num::Int: return static_cast<double>(n.i);
    case Num::Uint: return static_cast<double>(n.u);
    default: return n.f;
  }
}
uint64_t num_as_u64(const Num& n) {  // get<uint64_t>()
  switch (n.t) {
    case Num::Int: return static_cast<uint64_t>(n.i);
    case Num::Uint: return n.u;
    default: return static_cast<uint64_t>(n.f);
  }
}
int64_t num_as_i64(const Num& n) {  // get<int64_t>()
  switch (n.t) {
    case Num::Int: return n.i;
    case Num::Uint: return static_cast<int64_t>(n.u);
    default: return static_cast<int64_t>(n.f);
  }
}

// Decoded (escaped) strings of one worker thread; views into it stay valid
// (deque growth never moves elements) until the ingest returns.
struct Arena {
  std::deque<std::string> strings;
  std::string_view keep(const std::string& s) {
    strings.push_back(s);
    return std::string_view(strings.back());
  }
};

// an ArgMap value (trace.hpp ArgValue): string / bool / int64 / double
struct Arg {
  enum T : uint8_t { None, Str, Bool, Int, Dbl } t;
  bool b;
  int64_t i;
  double f;
  std::string_view s;  // into the document, or into the worker's arena
};

struct Keys {
  std::string fm = "forward_mode", batch = "batch_size", in = "input_len", out = "output_len";
};

// the args the path reads, after flattening (later writes win)
struct Args {
  Arg fm, batch, in, out, comm, rank, value, corr, host, dev, ref_ts;
  uint64_t dropped = 0;
  Arg* slot(std::string_view k, const Keys& keys) {
    using namespace std::string_view_literals;
    if (k == keys.fm) return &fm;
    if (k == keys.batch) return &batch;
    if (k == keys.in) return &in;
    if (k == keys.out) return &out;
    if (k == "commHash"sv) return &comm;
    if (k == "rank"sv) return &rank;
    if (k == "value"sv) return &value;
    if (k == "correlation_id"sv) return &corr;
    if (k == "hostname"sv) return &host;
    if (k == "device"sv) return &dev;
    if (k == "reference_ts"sv) return &ref_ts;
    return nullptr;
  }
};

// one scalar at s.p into *dst (null: dropped, counted)
void scalar(Scanner& s, Arg* dst, Args& a, Arena& arena) {
  const char c = s.peek();
  if (c == '"') {
    std::string buf;
    const std::string_view v = s.str_view(buf);
    if (dst) {
      dst->t = Arg::Str;
      dst->s = v.data() == buf.data() ? arena.keep(buf) : v;
    }
  } else if (c == 't') {
    s.literal("true");
    if (dst) {
      dst->t = Arg::Bool;
      dst->b = true;
    }
  } else if (c == 'f') {
    s.literal("false");
    if (dst) {
      dst->t = Arg::Bool;
      dst->b = false;
    }
  } else if (c == 'n') {
    s.literal("null");
    ++a.dropped;  // unsupported type: dropped with a warning
  } else {
    bool is_int = false;
    const std::string_view tok = s.number(&is_int);
    if (dst) {
      const Num n = parse_number(tok, is_int);
      if (n.t == Num::Float) {
        dst->t = Arg::Dbl;
        dst->f = n.f;
      } else {
        dst->t = Arg::Int;
        dst->i = num_as_i64(n);
      }
    }
  }
}

// flatten_args (trace_io.cpp:27-57) restricted to the keys the path reads;
// exact version: object members visited in key order after duplicate
// resolution (nlohmann objects are std::maps), arrays in order
void flatten(Scanner& s, const std::string& prefix, Args& a, const Keys& keys, Arena& arena) {
  const char c = s.peek();
  if (c == '{') {
    ++s.p;
    std::map<std::string, const char*> members;  // key -> value position (last wins)
    if (s.peek() != '}') {
      while (true) {
        std::string k;
        s.string(&k);
        s.expect(':');
        s.ws();
        members[k] = s.p;
        s.skip();
        const char d = s.peek();
        ++s.p;
        if (d == '}') break;
        if (d != ',') throw BadJson{};
      }
    } else {
      ++s.p;
    }
    const char* resume = s.p;
    for (const auto& [k, pos] : members) {
      Scanner sub{pos, s.end};
      flatten(sub, prefix.empty() ? k : prefix + "." + k, a, keys, arena);
    }
    s.p = resume;
    return;
  }
  if (c == '[') {
    ++s.p;
    size_t i = 0;
    if (s.peek() == ']') {
      ++s.p;
      return;
    }
    while (true) {
      flatten(s, prefix + "." + std::to_string(i++), a, keys, arena);
      const char d = s.peek();
      ++s.p;
      if (d == ']') return;
      if (d != ',') throw BadJson{};
    }
  }
  scalar(s, a.slot(prefix, keys), a, arena);
}

// args object: when every member is a scalar and no key contains '.', each
// member flattens to its own key, so document order with last-wins equals the
// sorted visit; otherwise the exact flatten above
void parse_args(const char* pos, const char* end, Args& a, const Keys& keys, Arena& arena) {
  Scanner s{pos, end};
  if (s.peek() == '{') {
    Scanner probe = s;
    ++probe.p;
    bool simple = true;
    if (probe.peek() != '}') {
      while (true) {
        std::string kb;
        const std::string_view k = probe.str_view(kb);
        if (k.find('.') != std::string_view::npos) simple = false;
        probe.expect(':');
        const char v = probe.peek();
        if (v == '{' || v == '[') simple = false;
        probe.skip();
        const char d = probe.peek();
        ++probe.p;
        if (d == '}') break;
        if (d != ',') throw BadJson{};
      }
    }
    if (simple) {
      ++s.p;
      if (s.peek() == '}') return;
      while (true) {
        std::string kb;
        const std::string_view k = s.str_view(kb);
        s.expect(':');
        scalar(s, a.slot(k, keys), a, arena);
        const char d = s.peek();
        ++s.p;
        if (d == '}') return;
      }
    }
  }
  flatten(s, "", a, keys, arena);
}

std::optional<int64_t> arg_int(const Arg& a) {  // trace.cpp:76-84
  if (a.t == Arg::Int) return a.i;
  if (a.t == Arg::Dbl) return static_cast<int64_t>(a.f);
  if (a.t == Arg::Bool) return a.b ? 1 : 0;
  return std::nullopt;
}
std::optional<double> arg_number(const Arg& a) {  // trace.cpp:86-93
  if (a.t == Arg::Dbl) return a.f;
  if (a.t == Arg::Int) return static_cast<double>(a.i);
  if (a.t == Arg::Bool) return a.b ? 1.0 : 0.0;
  return std::nullopt;
}
const std::string_view* arg_string(const Arg& a) { return a.t == Arg::Str ? &a.s : nullptr; }

// ------------------------------------------------------------ records
struct Rec {
  bool keep = false;
  // parse issues, in the order parse_record pushes them: a leading one that
  // ends the record (1 = not an event object / no "ph": error, 2 =
  // unsupported phase: warning), or an unknown-category warning, one
  // malformed_args warning per dropped args key, and a type error last
  uint8_t lead = 0;
  bool cat_warn = false, type_err = false;
  uint32_t dropped = 0;
  bool has_eid = false;
  uint64_t eid = 0;
  int kind = 0, category = 0;
  std::string_view name;  // into the document, or into the worker's arena
  std::string_view domain = "reference";  // source.clock_domain
  int64_t start = 0, dur = 0;
  Args args;
  uint32_t name_id = 0;
};

int kind_from_phase(std::string_view ph) {  // trace.cpp:44-50
  if (ph == "X") return CS_SPAN;
  if (ph == "i" || ph == "I") return CS_INSTANT;
  if (ph == "C") return CS_COUNTER;
  if (ph == "s" || ph == "f" || ph == "t") return CS_FLOW;
  return -1;
}
int category_from_string(std::string_view s) {  // trace.cpp:52-66
  static constexpr std::string_view kNames[] = {"python_call", "runtime_api", "gpu_kernel",
                                                "mem_copy",    "os_sched",    "net_io",
                                                "counter_telemetry", "collective_comm"};
  for (int i = 0; i < 8; ++i)
    if (s == kNames[i]) return i;
  return -1;
}
int64_t us_to_ns(double us) { return static_cast<int64_t>(std::llround(us * 1000.0)); }

// typed access to a value at a validated position (type errors drop the record)
std::string_view as_string(const char* pos, const char* end, std::string& buf) {
  Scanner s{pos, end};
  if (s.peek() != '"') throw TypeError{};
  return s.str_view(buf);
}
Num as_number(const char* pos, const char* end) {
  Scanner s{pos, end};
  const char c = s.peek();
  if (c != '-' && (c < '0' || c > '9')) throw TypeError{};
  bool is_int = false;
  const std::string_view tok = s.number(&is_int);
  return parse_number(tok, is_int);
}

// parse_record (trace_io.cpp:87-158) on one object: a single validating pass
// over its members (the last occurrence of a key wins), then typed reads in
// the reference's order
void parse_record(const char* b, const char* e, Rec& r, const Keys& keys, Arena& arena) {
  Scanner s{b, e};
  if (s.peek() != '{') {
    s.skip();
    s.ws();
    if (s.p != s.end) throw BadJson{};
    r.lead = 1;  // "record is not an event object"
    return;
  }
  ++s.p;
  enum { kPh, kEid, kName, kTs, kDur, kPid, kTid, kCat, kSrc, kArgs, kN };
  static constexpr std::string_view kKeys[kN] = {"ph",  "eid", "name", "ts",  "dur",
                                                 "pid", "tid", "cat",  "src", "args"};
  const char* pos[kN] = {};
  if (s.peek() != '}') {
    std::string kb;
    while (true) {
      const std::string_view k = s.str_view(kb);
      s.expect(':');
      s.ws();
      if (k.size() <= 4)
        for (int i = 0; i < kN; ++i)
          if (k == kKeys[i]) pos[i] = s.p;
      s.skip();
      const char d = s.peek();
      ++s.p;
      if (d == '}') break;
      if (d != ',') throw BadJson{};
    }
  } else {
    ++s.p;
  }
  s.ws();
  if (s.p != s.end) throw BadJson{};  // spans come from the parallel splitter, untrimmed
  try {
    if (!pos[kPh]) {
      r.lead = 1;
      return;
    }
    std::string buf;
    const std::string_view ph = as_string(pos[kPh], e, buf);
    if (ph == "M") return;
    r.kind = kind_from_phase(ph);
    if (r.kind < 0) {
      r.lead = 2;
      return;
    }
    if (pos[kEid]) {
      r.has_eid = true;
      r.eid = num_as_u64(as_number(pos[kEid], e));
    }
    if (pos[kName]) {
      const std::string_view n = as_string(pos[kName], e, buf);
      r.name = n.data() == buf.data() ? arena.keep(buf) : n;
    }
    double ts = 0.0, dur = 0.0;
    if (pos[kTs]) ts = num_as_double(as_number(pos[kTs], e));
    r.start = us_to_ns(ts);
    if (r.kind == CS_SPAN) {
      if (pos[kDur]) dur = num_as_double(as_number(pos[kDur], e));
      r.dur = us_to_ns(dur);
    }
    if (pos[kPid]) as_number(pos[kPid], e);
    if (pos[kTid]) as_number(pos[kTid], e);
    r.category = r.kind == CS_COUNTER ? CS_CAT_COUNTER_TELEMETRY : CS_CAT_PYTHON_CALL;
    if (pos[kCat]) {
      const int c = category_from_string(as_string(pos[kCat], e, buf));
      if (c < 0) r.cat_warn = true;  // unknown category: warning, default kept
      else r.category = c;
    }
    if (pos[kSrc]) {
      Scanner ss{pos[kSrc], e};
      if (ss.peek() == '{') {  // node / clock / collector must be strings when present
        ++ss.p;
        if (ss.peek() != '}') {
          const char* sp[3] = {};
          while (true) {
            const std::string_view k = ss.str_view(buf);
            const int i = k == "node" ? 0 : k == "clock" ? 1 : k == "collector" ? 2 : -1;
            ss.expect(':');
            ss.ws();
            if (i >= 0) sp[i] = ss.p;
            ss.skip();
            const char d = ss.peek();
            ++ss.p;
            if (d == '}') break;
          }
          for (const char* q : sp)
            if (q) as_string(q, e, buf);
          if (sp[1]) {
            const std::string_view v = as_string(sp[1], e, buf);
            r.domain = v.data() == buf.data() ? arena.keep(buf) : v;
          }
        }
      }
    }
    if (pos[kArgs]) {
      parse_args(pos[kArgs], e, r.args, keys, arena);
      r.dropped = static_cast<uint32_t>(r.args.dropped);
    }
    r.keep = true;
  } catch (const TypeError&) {
    r.keep = false;
    r.type_err = true;
  }
}

using cs_host::parallel_for;

// Split the array whose '[' is at a into element spans, in parallel; returns
// one past its ']'.  Two passes over fixed chunks of the remaining text:
// (1) the parity of unescaped quotes per chunk (backslashes are treated as
// escapes everywhere: outside strings they are invalid JSON, and a document
// that holds one is rejected by the per-span parse whatever the split), a
// prefix of which gives each chunk's string state at its start; (2) per chunk,
// the commas and closing brackets met at the running minimum of the relative
// depth.  A prefix over the chunks' depth changes then keeps the commas at
// array depth and the first bracket that closes the array.  Chunk starts are
// moved past backslashes so no chunk begins on an escaped character.
// Element validity is left to the record parser (a concatenation of valid
// values separated by commas is a valid array, so the split cannot hide an
// error).
const char* split_array(const char* a, const char* end, uint32_t n_threads,
                        std::vector<std::pair<const char*, const char*>>& spans) {
  const char* r0 = a + 1;
  const size_t len = static_cast<size_t>(end - r0);
  const uint32_t nc = static_cast<uint32_t>(
      std::max<size_t>(1, std::min<size_t>(n_threads * 4u, len / (1u << 16))));
  std::vector<const char*> cb(nc + 1);
  cb[0] = r0;
  cb[nc] = end;
  for (uint32_t c = 1; c < nc; ++c) {
    const char* q = std::max(cb[c - 1], r0 + len * c / nc);
    while (q < end && q > r0 && q[-1] == '\\') ++q;
    cb[c] = q;
  }
  // pass 1: quote parity
  std::vector<uint8_t> par(nc + 1, 0);
  parallel_for(nc, n_threads, [&](size_t c0, size_t c1, uint32_t) {
    for (size_t c = c0; c < c1; ++c) {
      const char* q = cb[c];
      const char* e = cb[c + 1];
      uint8_t x = 0;
      while (true) {
        q = Scanner::next_quote(q, e);
        if (q >= e) break;
        if (*q == '\\') {
          q += 2;
        } else {
          x ^= 1;
          ++q;
        }
      }
      par[c + 1] = x;
    }
  });
  for (uint32_t c = 0; c < nc; ++c) par[c + 1] ^= par[c];
  // pass 2: candidates at the running minimum depth
  struct Cand {
    const char* p;
    int depth;  // relative depth after the character
    char ch;
  };
  std::vector<std::vector<Cand>> cand(nc);
  std::vector<int> delta(nc, 0);
  parallel_for(nc, n_threads, [&](size_t c0, size_t c1, uint32_t) {
    for (size_t c = c0; c < c1; ++c) {
      const char* q = cb[c];
      const char* e = cb[c + 1];
      bool in_str = par[c];
      int d = 0, lo = 0;
      auto& out = cand[c];
      while (q < e) {
        if (in_str) {
          q = Scanner::next_quote(q, e);
          if (q >= e) break;
          if (*q == '\\') {
            q += 2;
            continue;
          }
          in_str = false;
          ++q;
          continue;
        }
        q = Scanner::next_special_comma(q, e);
        if (q >= e) break;
        const char x = *q;
        if (x == '"') {
          in_str = true;
        } else if (x == '{' || x == '[') {
          ++d;
        } else if (x == ',') {
          if (d <= lo) out.push_back({q, d, x});
        } else if (x == '}' || x == ']') {
          --d;
          if (d <= lo) {
            lo = d;
            out.push_back({q, d, x});
          }
        } else {  // backslash outside a string: invalid, the span parse rejects it
          ++q;
        }
        ++q;
      }
      delta[c] = d;
    }
  });
  // sequential: absolute depth 1 = inside the array
  const char* b = r0;
  int d0 = 1;
  for (uint32_t c = 0; c < nc; ++c) {
    for (const Cand& k : cand[c]) {
      const int d = d0 + k.depth;
      if (k.ch == ',' && d == 1) {
        spans.emplace_back(b, k.p);
        b = k.p + 1;
      } else if (d == 0) {
        if (k.ch != ']') throw BadJson{};
        // an empty array is the only place an empty element is allowed
        const char* t = b;
        while (t < k.p && (*t == ' ' || *t == '\t' || *t == '\n' || *t == '\r')) ++t;
        if (t != k.p || !spans.empty()) spans.emplace_back(b, k.p);
        return k.p + 1;
      }
    }
    d0 += delta[c];
  }
  throw BadJson{};  // unterminated array
}

// validate_trace (trace.cpp:239-276) over the canonical record order: per
// event a duplicate id (at its second occurrence), a negative span duration,
// a non-span duration; then check_correlations (158-201) and check_counters
// (203-235).  Duplicate ids are found in parallel (one hash partition of the
// ids per thread, all scanning in event order) unless the ids increase.
void validate(cs_ingest_result& res, const std::vector<std::pair<size_t, uint64_t>>& corr,
              uint32_t n_threads) {
  const size_t n = res.events.size();
  const uint64_t* ids = res.event_ids.data();
  for (const cs_event& e : res.events) ++res.categories[e.category & 7];
  std::vector<uint8_t> dup2(n, 0);
  bool increasing = true;
  uint64_t lo = n ? ids[0] : 0, hi = lo;
  for (size_t i = 1; i < n; ++i) {
    increasing = increasing && ids[i] > ids[i - 1];
    lo = std::min(lo, ids[i]);
    hi = std::max(hi, ids[i]);
  }
  if (!increasing) {
    // each thread owns a slice of the id space and scans every event in order
    const bool dense = hi - lo < 8 * static_cast<uint64_t>(n) + 64;
    parallel_for(n_threads, n_threads, [&](size_t t0, size_t t1, uint32_t) {
      for (size_t t = t0; t < t1; ++t) {
        if (dense) {
          const uint64_t span = hi - lo + 1;
          const uint64_t a = lo + span * t / n_threads, b = lo + span * (t + 1) / n_threads;
          std::vector<uint64_t> once((b - a + 63) / 64, 0), twice((b - a + 63) / 64, 0);
          for (size_t i = 0; i < n; ++i) {
            const uint64_t x = ids[i];
            if (x < a || x >= b) continue;
            const uint64_t k = x - a, w = k >> 6, m = 1ull << (k & 63);
            if (!(once[w] & m)) {
              once[w] |= m;
            } else if (!(twice[w] & m)) {
              twice[w] |= m;
              dup2[i] = 1;
            }
          }
        } else {
          std::unordered_map<uint64_t, uint32_t> seen;
          for (size_t i = 0; i < n; ++i) {
            if ((ids[i] * 0x9E3779B97F4A7C15ull >> 40) % n_threads != t) continue;
            if (++seen[ids[i]] == 2) dup2[i] = 1;
          }
        }
      }
    });
  }
  for (size_t i = 0; i < n; ++i) {
    const cs_event& e = res.events[i];
    if (dup2[i]) res.issue(CS_SEV_ERROR, CS_ISSUE_DUPLICATE_EVENT_ID, true, ids[i]);
    if (e.kind == CS_SPAN && e.duration < 0)
      res.issue(CS_SEV_ERROR, CS_ISSUE_NEGATIVE_DURATION, true, ids[i]);
    if (e.kind != CS_SPAN && e.kind != CS_COUNTER && e.duration != 0)
      res.issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_EVENT, true, ids[i]);
  }
  // correlations: host side = RuntimeApi, device side = GpuKernel / MemCopy
  if (!corr.empty()) {
    std::unordered_map<uint64_t, int> host, device;
    auto is_dev = [&](size_t i) {
      return res.events[i].category == CS_CAT_GPU_KERNEL || res.events[i].category == CS_CAT_MEM_COPY;
    };
    for (const auto& [i, c] : corr) {
      if (res.events[i].category == CS_CAT_RUNTIME_API) ++host[c];
      else if (is_dev(i)) ++device[c];
    }
    for (const auto& [i, c] : corr) {
      if (is_dev(i)) {
        if (device[c] > 1) res.issue(CS_SEV_ERROR, CS_ISSUE_DUPLICATE_CORRELATION, true, ids[i]);
        else if (!host.count(c)) res.issue(CS_SEV_WARNING, CS_ISSUE_UNMATCHED_CORRELATION, true, ids[i]);
      } else if (res.events[i].category == CS_CAT_RUNTIME_API && host[c] > 1) {
        res.issue(CS_SEV_ERROR, CS_ISSUE_DUPLICATE_CORRELATION, true, ids[i]);
      }
    }
  }
  // counters: a numeric, finite value; strictly increasing ts per series name
  std::vector<int64_t> last(res.n_names, 0);
  std::vector<uint8_t> has_last(res.n_names, 0), flagged(res.n_names, 0);
  for (size_t i = 0; i < n; ++i) {
    const cs_event& e = res.events[i];
    if (e.kind != CS_COUNTER) continue;
    if (!(e.flags & CS_EV_HAS_VALUE)) {
      res.issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_ARGS, true, ids[i]);
      continue;
    }
    double v;
    std::memcpy(&v, &e.duration, sizeof v);
    if (!std::isfinite(v)) res.issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_ARGS, true, ids[i]);
    const uint32_t k = e.name_id;
    if (has_last[k] && e.start_ts <= last[k] && !flagged[k]) {
      res.issue(CS_SEV_ERROR, CS_ISSUE_NON_MONOTONE_COUNTER, true, ids[i]);
      flagged[k] = 1;
    }
    last[k] = e.start_ts;
    has_last[k] = 1;
  }
}

struct CommKey {
  std::string_view name, hash;
  int rank;
  bool operator<(const CommKey& o) const {
    if (name != o.name) return name < o.name;
    if (hash != o.hash) return hash < o.hash;
    return rank < o.rank;
  }
  bool operator==(const CommKey& o) const { return name == o.name && hash == o.hash && rank == o.rank; }
};

}  // namespace

extern "C" {

static int cs_ingest_chrome_json_impl(const char* text, size_t len, const cs_ingest_keys* keys_in,
                          uint32_t n_threads, cs_ingest_result** out) {
  if (!out || (len && !text)) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  Keys keys;
  if (keys_in) {
    if (keys_in->forward_mode) keys.fm = keys_in->forward_mode;
    if (keys_in->batch_size) keys.batch = keys_in->batch_size;
    if (keys_in->input_len) keys.in = keys_in->input_len;
    if (keys_in->output_len) keys.out = keys_in->output_len;
  }
  if (n_threads == 0) n_threads = 1;
  auto* res = new cs_ingest_result();
  auto reject = [&]() {
    res->n_issues = 1;  // parse_error: empty trace, one issue
    res->issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_EVENT, false, 0);
    *out = res;
    return CS_OK;
  };
  // ---- locate the events array and split it into records
  std::vector<std::pair<const char*, const char*>> spans;
  try {
    Scanner s{text, text + len};
    const char* arr = nullptr;
    const char* arr_end = nullptr;
    const char c = s.peek();
    bool not_events = false;
    if (c == '[') {
      arr = s.p;
      arr_end = split_array(arr, s.end, n_threads, spans);
      s.p = arr_end;
      s.ws();
      if (s.p != s.end) throw BadJson{};
    } else if (c == '{') {
      ++s.p;
      if (s.peek() != '}') {
        while (true) {
          std::string k;
          s.string(&k);
          s.expect(':');
          s.ws();
          const char* v = s.p;
          if (k == "traceEvents" && *v == '[') {
            if (arr) {  // superseded (nlohmann keeps the last): still validated
              Scanner old{arr, arr_end};
              old.skip();
            }
            spans.clear();  // split here, validated by the record parsers
            s.p = split_array(v, s.end, n_threads, spans);
            arr = v;
            arr_end = s.p;
          } else {
            if (k == "traceEvents" && arr) {
              Scanner old{arr, arr_end};
              old.skip();
              arr = nullptr, arr_end = nullptr;
              spans.clear();
            }
            s.skip();
          }
          const char d = s.peek();
          ++s.p;
          if (d == '}') break;
          if (d != ',') throw BadJson{};
        }
      } else {
        ++s.p;
      }
      s.ws();
      if (s.p != s.end) throw BadJson{};
      not_events = arr == nullptr;
    } else {
      s.skip();
      s.ws();
      if (s.p != s.end) throw BadJson{};
      not_events = true;
    }
    if (not_events) {
      res->n_issues = 1;  // neither an event array nor an object with traceEvents
      res->issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_EVENT, false, 0);
      *out = res;
      return CS_OK;
    }
  } catch (const BadJson&) {
    return reject();
  }
  // ---- records in parallel (a syntax error anywhere rejects the document)
  // records live in per-thread chunks (first touch by their worker)
  std::vector<std::vector<Rec>> chunks(n_threads);
  std::vector<size_t> chunk0(n_threads + 1, 0);
  for (uint32_t t = 0; t <= n_threads; ++t) chunk0[t] = spans.size() * t / n_threads;
  auto rec = [&](size_t k) -> Rec& {
    const uint32_t t = static_cast<uint32_t>(
        std::upper_bound(chunk0.begin(), chunk0.end(), k) - chunk0.begin() - 1);
    return chunks[t][k - chunk0[t]];
  };
  std::vector<uint8_t> bad(n_threads, 0);
  std::vector<Arena> arenas(n_threads);
  parallel_for(spans.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
    chunks[t].resize(k1 - k0);
    try {
      for (size_t k = k0; k < k1; ++k)
        parse_record(spans[k].first, spans[k].second, chunks[t][k - k0], keys, arenas[t]);
    } catch (const BadJson&) {
      bad[t] = 1;
    }
  });
  for (uint8_t x : bad)
    if (x) return reject();
  // ---- fallback ids in document order, then the canonical stable sort.
  // next_id evolves as x -> max(x, eid) + 1 per kept record (a fallback id is
  // x itself), i.e. x -> max(x + a, b): such maps compose, so each chunk's map
  // is built in parallel, chained sequentially (one per chunk), and the ids
  // assigned in parallel.  A chunk holding an id that could wrap the uint64
  // arithmetic is done sequentially instead (the reference wraps too).
  const uint32_t nchunk = n_threads;
  struct Affine {
    uint64_t a = 0, b = 0;  // x -> max(x + a, b); b = 0 is "no bound" (x >= 1)
    bool wraps = false;
  };
  std::vector<Affine> maps(nchunk);
  parallel_for(nchunk, nchunk, [&](size_t t0, size_t t1, uint32_t) {
    for (size_t t = t0; t < t1; ++t) {
      Affine m;
      for (const Rec& r : chunks[t]) {
        if (!r.keep) continue;
        if (r.has_eid && r.eid >= (UINT64_MAX >> 1)) m.wraps = true;
        m.b = r.has_eid ? std::max(m.b + 1, r.eid + 1) : m.b + 1;
        m.a += 1;
      }
      maps[t] = m;
    }
  });
  bool any_wrap = false;
  for (const auto& m : maps) any_wrap |= m.wraps;
  std::vector<uint64_t> next_in(nchunk + 1, 1);
  for (uint32_t t = 0; t < nchunk && !any_wrap; ++t)
    next_in[t + 1] = std::max(next_in[t] + maps[t].a, maps[t].b);
  // per chunk: ids, parse issues (with the id each record had at its turn), kept records
  std::vector<std::vector<cs_ingest_issue>> tiss(nchunk);
  std::vector<std::vector<Rec*>> tkept(nchunk);
  auto chunk_ids = [&](uint32_t t, uint64_t& next_id) {
    auto issue = [&](uint8_t sev, uint8_t code, bool has_id, uint64_t id) {
      cs_ingest_issue x{};
      x.severity = sev;
      x.code = code;
      x.has_event_id = has_id ? 1 : 0;
      x.event_id = has_id ? id : 0;
      tiss[t].push_back(x);
    };
    tkept[t].reserve(chunks[t].size());
    for (Rec& r : chunks[t]) {
      const uint64_t id_now = r.has_eid ? r.eid : next_id;
      if (r.lead) {
        issue(r.lead == 1 ? CS_SEV_ERROR : CS_SEV_WARNING, CS_ISSUE_MALFORMED_EVENT, false, 0);
      } else {
        if (r.cat_warn) issue(CS_SEV_WARNING, CS_ISSUE_MALFORMED_EVENT, true, id_now);
        for (uint32_t q = 0; q < r.dropped; ++q) issue(CS_SEV_WARNING, CS_ISSUE_MALFORMED_ARGS, true, id_now);
        if (r.type_err) issue(CS_SEV_ERROR, CS_ISSUE_MALFORMED_EVENT, false, 0);
      }
      if (!r.keep) continue;
      if (!r.has_eid) r.eid = next_id;
      next_id = std::max(next_id, r.eid) + 1;
      tkept[t].push_back(&r);
    }
  };
  if (any_wrap) {
    uint64_t next_id = 1;
    for (uint32_t t = 0; t < nchunk; ++t) chunk_ids(t, next_id);
  } else {
    parallel_for(nchunk, nchunk, [&](size_t t0, size_t t1, uint32_t) {
      for (size_t t = t0; t < t1; ++t) {
        uint64_t next_id = next_in[t];
        chunk_ids(static_cast<uint32_t>(t), next_id);
      }
    });
  }
  std::vector<Rec*> kept;
  {
    size_t nk = 0;
    for (const auto& v : tkept) nk += v.size();
    kept.reserve(nk);
  }
  for (uint32_t t = 0; t < nchunk; ++t) {
    for (const auto& x : tiss[t]) res->issue(x.severity, x.code, x.has_event_id != 0, x.event_id);
    kept.insert(kept.end(), tkept[t].begin(), tkept[t].end());
  }
  (void)rec;
  {
    struct Key {
      int64_t start;
      uint64_t eid;
      Rec* idx;
    };
    auto less = [](const Key& a, const Key& b) {
      return a.start != b.start ? a.start < b.start : a.eid < b.eid;
    };
    std::vector<Key> keys_v(kept.size());
    std::vector<uint8_t> unsorted(n_threads, 0);
    parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
      for (size_t i = k0; i < k1; ++i) keys_v[i] = {kept[i]->start, kept[i]->eid, kept[i]};
      for (size_t i = k0 + 1; i < k1 && !unsorted[t]; ++i) unsorted[t] = less(keys_v[i], keys_v[i - 1]);
    });
    bool sorted = true;
    for (uint8_t u : unsorted) sorted = sorted && !u;
    if (sorted)  // chunk boundaries
      for (uint32_t t = 1; t < n_threads && sorted; ++t) {
        const size_t i = kept.size() * t / std::max<size_t>(1, std::min<size_t>(n_threads, kept.size() ? kept.size() : 1));
        if (i > 0 && i < kept.size()) sorted = !less(keys_v[i], keys_v[i - 1]);
      }
    if (!sorted) {
      std::stable_sort(keys_v.begin(), keys_v.end(), less);
      for (size_t i = 0; i < kept.size(); ++i) kept[i] = keys_v[i].idx;
    }
  }
  // ---- interning: names and (name, commHash, rank) in sorted order
  std::vector<std::vector<std::string_view>> tn(n_threads);
  std::vector<std::vector<CommKey>> tc(n_threads);
  parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
    std::unordered_set<std::string_view> seen;
    std::set<CommKey> cs;
    for (size_t k = k0; k < k1; ++k) {
      const Rec& r = *kept[k];
      seen.insert(r.name);
      if (r.kind == CS_SPAN && r.category == CS_CAT_COLLECTIVE_COMM) {
        const std::string_view* comm = arg_string(r.args.comm);
        const auto rank = arg_int(r.args.rank);
        if (comm && rank) cs.insert({r.name, *comm, static_cast<int>(*rank)});
      }
    }
    tn[t].assign(seen.begin(), seen.end());
    tc[t].assign(cs.begin(), cs.end());
  });
  std::vector<std::string_view> names;
  std::vector<CommKey> comms;
  for (uint32_t t = 0; t < n_threads; ++t) {
    names.insert(names.end(), tn[t].begin(), tn[t].end());
    comms.insert(comms.end(), tc[t].begin(), tc[t].end());
  }
  std::sort(names.begin(), names.end());
  names.erase(std::unique(names.begin(), names.end()), names.end());
  std::sort(comms.begin(), comms.end());
  comms.erase(std::unique(comms.begin(), comms.end()), comms.end());
  std::unordered_map<std::string_view, uint32_t> name_id;
  for (uint32_t i = 0; i < names.size(); ++i) {
    name_id[names[i]] = i;
    res->names_packed.append(names[i]);
    res->names_packed.push_back('\0');
  }
  res->n_names = static_cast<uint32_t>(names.size());
  for (const auto& ck : comms) {
    res->comm_name.push_back(static_cast<int32_t>(name_id[ck.name]));
    res->comm_rank.push_back(ck.rank);
    res->comm_hash_packed.append(ck.hash);
    res->comm_hash_packed.push_back('\0');
  }
  // ---- topology: (commHash, rank) -> (hostname, device) from every
  // CollectiveComm record carrying all four args; a key mapped to two
  // locations is the reference's ConflictingTopology
  {
    using Key = std::pair<std::string_view, int>;
    using Loc = std::pair<std::string_view, int>;
    std::vector<std::vector<std::pair<Key, Loc>>> tl(n_threads);
    parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
      for (size_t k = k0; k < k1; ++k) {
        const Rec& r = *kept[k];
        if (r.category != CS_CAT_COLLECTIVE_COMM) continue;
        const std::string_view* comm = arg_string(r.args.comm);
        const std::string_view* host = arg_string(r.args.host);
        const auto rank = arg_int(r.args.rank), dev = arg_int(r.args.dev);
        if (comm && rank && host && dev)
          tl[t].push_back({{*comm, static_cast<int>(*rank)}, {*host, static_cast<int>(*dev)}});
      }
    });
    std::map<Key, Loc> topo;
    for (const auto& v : tl)
      for (const auto& [key, loc] : v) {
        const auto [it, inserted] = topo.emplace(key, loc);
        if (!inserted && it->second != loc) res->topology_conflict = 1;
      }
    for (const auto& [key, loc] : topo)
      res->topo.emplace_back(std::string(key.first), key.second, std::string(loc.first), loc.second);
    std::vector<Loc> locs;
    for (const auto& kv : topo) locs.push_back(kv.second);
    std::sort(locs.begin(), locs.end());
    locs.erase(std::unique(locs.begin(), locs.end()), locs.end());
    for (const auto& l : locs) {
      res->loc_nodes_packed.append(l.first);
      res->loc_nodes_packed.push_back('\0');
      res->loc_device.push_back(l.second);
    }
    for (const auto& ck : comms) {
      const auto it = topo.find({ck.hash, ck.rank});
      res->comm_location.push_back(
          it == topo.end() ? -1
                           : static_cast<int32_t>(std::lower_bound(locs.begin(), locs.end(), it->second) - locs.begin()));
    }
  }
  // ---- records (the exporters' contract, include/cyclescope_b200.h)
  res->events.resize(kept.size());
  res->event_ids.resize(kept.size());
  std::vector<uint8_t> carries(kept.size(), 0);
  // correlation ids (integer args.correlation_id, trace_io.cpp:151-156), per worker in order
  std::vector<std::vector<std::pair<size_t, uint64_t>>> tcorr(n_threads);
  parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
    for (size_t i = k0; i < k1; ++i) {
      const Rec& r = *kept[i];
      if (r.args.corr.t == Arg::Int) tcorr[t].push_back({i, static_cast<uint64_t>(r.args.corr.i)});
      cs_event& o = res->events[i];
      std::memset(&o, 0, sizeof o);
      o.start_ts = r.start;
      o.duration = r.kind == CS_SPAN ? r.dur : 0;
      o.name_id = name_id.at(r.name);
      o.kind = static_cast<uint8_t>(r.kind);
      o.category = static_cast<uint8_t>(r.category);
      uint16_t flags = 0;
      if (const std::string_view* fm = arg_string(r.args.fm)) {  // cycles.cpp:205-220
        std::string m(*fm);
        for (auto& ch : m) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
        if (m.find("prefill") != std::string::npos || m.find("extend") != std::string::npos)
          flags |= CS_EV_FM_PREFILL;
        else if (m.find("decode") != std::string::npos)
          flags |= CS_EV_FM_DECODE;
        else
          flags |= CS_EV_FM_OTHER;
      }
      if (const auto b = arg_int(r.args.batch)) {  // cycles.cpp:256-281
        flags |= CS_EV_HAS_BATCH;
        const auto in = arg_int(r.args.in), ou = arg_int(r.args.out);
        if (in && ou && *b >= 0 && *in >= 0 && *ou >= 0) flags |= CS_EV_WL_OK;
        carries[i] = 1;
      }
      if (r.kind == CS_SPAN && r.category == CS_CAT_COLLECTIVE_COMM) {  // rca.cpp:108-115
        const std::string_view* comm = arg_string(r.args.comm);
        const auto rank = arg_int(r.args.rank);
        if (comm && rank) {
          flags |= CS_EV_HAS_COMM;
          const CommKey ck{r.name, *comm, static_cast<int>(*rank)};
          const auto it = std::lower_bound(comms.begin(), comms.end(), ck);
          o.payload |= static_cast<uint64_t>(it - comms.begin()) << 32;
        }
      }
      if (r.kind == CS_COUNTER) {
        if (const auto v = arg_number(r.args.value)) {
          flags |= CS_EV_HAS_VALUE;
          std::memcpy(&o.duration, &*v, sizeof(double));
        }
      }
      o.flags = flags;
      res->event_ids[i] = r.eid;
    }
  });
  // workload table in event order (payload low 32 bits = its index)
  for (size_t i = 0; i < kept.size(); ++i) {
    if (!carries[i]) continue;
    const Rec& r = *kept[i];
    const auto b = arg_int(r.args.batch), in = arg_int(r.args.in), ou = arg_int(r.args.out);
    res->events[i].payload |= static_cast<uint64_t>(res->workloads.size());
    res->workloads.push_back({*b, in ? *in : INT64_MIN, ou ? *ou : INT64_MIN});
  }
  // clock domains (interned in name order) and inline beacons, in event order
  {
    std::vector<std::unordered_set<std::string_view>> td(n_threads);
    std::vector<std::vector<std::pair<uint64_t, int64_t>>> tb(n_threads);
    parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t t) {
      for (size_t k = k0; k < k1; ++k) {
        const Rec& r = *kept[k];
        td[t].insert(r.domain);
        if (r.kind == CS_INSTANT && r.name == "beacon")
          if (const auto ref = arg_int(r.args.ref_ts)) tb[t].push_back({k, *ref});
      }
    });
    std::set<std::string_view> ds;
    for (const auto& v : td) ds.insert(v.begin(), v.end());
    std::unordered_map<std::string_view, uint16_t> did;
    for (const auto& d : ds) {
      did[d] = static_cast<uint16_t>(res->domains.size());
      res->domains.emplace_back(d);
    }
    res->domain.resize(kept.size());
    parallel_for(kept.size(), n_threads, [&](size_t k0, size_t k1, uint32_t) {
      for (size_t k = k0; k < k1; ++k) res->domain[k] = did.at(kept[k]->domain);
    });
    for (const auto& v : tb) res->beacons.insert(res->beacons.end(), v.begin(), v.end());
  }
  res->n_issues = res->issues.size();
  std::vector<std::pair<size_t, uint64_t>> corr;
  for (const auto& v : tcorr) corr.insert(corr.end(), v.begin(), v.end());
  validate(*res, corr, n_threads);
  *out = res;
  return CS_OK;
}

int cs_ingest_chrome_json(const char* text, size_t len, const cs_ingest_keys* keys_in,
                          uint32_t n_threads, cs_ingest_result** out) {
  return cs_guard([&] { return cs_ingest_chrome_json_impl(text, len, keys_in, n_threads, out); });
}

int cs_ingest_view(const cs_ingest_result* r, const cs_event** ev, const uint64_t** event_ids,
                   uint64_t* n_ev, const cs_workload** wl, uint64_t* n_wl, const char** names,
                   size_t* names_bytes, uint32_t* n_names, const int32_t** comm_name,
                   const int32_t** comm_rank, const char** comm_hash, size_t* comm_bytes,
                   uint32_t* n_comm, uint64_t* n_issues) {
  if (!r) return CS_E_INVALID_ARGUMENT;
  if (ev) *ev = r->events.data();
  if (event_ids) *event_ids = r->event_ids.data();
  if (n_ev) *n_ev = r->events.size();
  if (wl) *wl = r->workloads.data();
  if (n_wl) *n_wl = r->workloads.size();
  if (names) *names = r->names_packed.data();
  if (names_bytes) *names_bytes = r->names_packed.size();
  if (n_names) *n_names = r->n_names;
  if (comm_name) *comm_name = r->comm_name.data();
  if (comm_rank) *comm_rank = r->comm_rank.data();
  if (comm_hash) *comm_hash = r->comm_hash_packed.data();
  if (comm_bytes) *comm_bytes = r->comm_hash_packed.size();
  if (n_comm) *n_comm = static_cast<uint32_t>(r->comm_name.size());
  if (n_issues) *n_issues = r->n_issues;
  return CS_OK;
}

static int cs_ingest_merge_impl(const cs_ingest_result* const* in, uint32_t n_in, const cs_calibration_options* opt,
                    uint32_t n_threads, cs_ingest_result** out, char* err, size_t err_cap) {
  if (!out || (n_in && !in)) return CS_E_INVALID_ARGUMENT;
  *out = nullptr;
  for (uint32_t t = 0; t < n_in; ++t)
    if (!in[t]) return CS_E_INVALID_ARGUMENT;
  if (n_threads == 0) n_threads = 1;
  auto failure = [&](int code, const std::string& msg) {
    if (err && err_cap) {
      std::strncpy(err, msg.c_str(), err_cap - 1);
      err[err_cap - 1] = 0;
    }
    return code;
  };
  // ---- calibrate (align.cpp:22-84) from every input's beacons, input order
  const std::string ref_dom = opt && opt->reference_domain ? opt->reference_domain : "reference";
  const double tol = opt ? opt->tolerance_ns : 1000.0;
  const bool fit_drift = opt && opt->estimate_drift;
  struct Beacon {
    std::string_view domain;
    int64_t local, ref;
  };
  std::map<std::string_view, std::vector<Beacon>> groups;
  for (uint32_t t = 0; t < n_in; ++t)
    for (const auto& [i, ref] : in[t]->beacons) {
      const std::string_view d = in[t]->domains[in[t]->domain[i]];
      if (d != ref_dom) groups[d].push_back({d, in[t]->events[i].start_ts, ref});
    }
  struct Clock {
    double offset = 0.0, drift = 1.0;
    bool identity() const { return offset == 0.0 && drift == 1.0; }
  };
  std::map<std::string, Clock, std::less<>> clocks;
  clocks[ref_dom] = Clock{};
  for (const auto& [dom, g] : groups) {
    Clock c;
    const double n = static_cast<double>(g.size());
    if (g.size() == 1) {
      c.offset = static_cast<double>(g[0].ref - g[0].local);
    } else if (!fit_drift) {
      double sum = 0.0;
      for (const auto& b : g) sum += static_cast<double>(b.ref - b.local);
      c.offset = sum / n;
    } else {  // least squares: ref = offset + drift * local
      double ml = 0.0, mr = 0.0;
      for (const auto& b : g) {
        ml += static_cast<double>(b.local);
        mr += static_cast<double>(b.ref);
      }
      ml /= n;
      mr /= n;
      double cov = 0.0, var = 0.0;
      for (const auto& b : g) {
        const double dl = static_cast<double>(b.local) - ml, dr = static_cast<double>(b.ref) - mr;
        cov += dl * dr;
        var += dl * dl;
      }
      c.drift = var > 0.0 ? cov / var : 1.0;
      c.offset = mr - c.drift * ml;
    }
    double worst = 0.0;
    for (const auto& b : g)
      worst = std::max(worst, std::abs(c.offset + c.drift * static_cast<double>(b.local) - static_cast<double>(b.ref)));
    if (worst > tol)
      return failure(CS_E_INCONSISTENT_BEACONS, "domain '" + std::string(dom) + "' max beacon residual " +
                                                    std::to_string(worst) + " ns exceeds tolerance");
    clocks[std::string(dom)] = c;
  }
  // ---- apply_calibration per input (align.cpp:97-113), then merge_traces (193-206)
  struct Item {
    int64_t ts;
    uint64_t eid;
    uint32_t t;
    uint64_t i;
  };
  std::vector<std::vector<Item>> items(n_in);
  std::vector<std::vector<cs_event>> evs(n_in);
  for (uint32_t t = 0; t < n_in; ++t) {
    const cs_ingest_result& r = *in[t];
    if (r.calibrated) return failure(CS_E_ALREADY_CALIBRATED, "trace timestamps are already on the unified timeline");
    std::vector<const Clock*> of(r.domains.size(), nullptr);
    for (size_t d = 0; d < r.domains.size(); ++d) {
      const auto it = clocks.find(r.domains[d]);
      if (it != clocks.end()) of[d] = &it->second;
    }
    for (size_t i = 0; i < r.events.size(); ++i)
      if (!of[r.domain[i]])
        return failure(CS_E_NO_BEACONS, "no calibration for clock domain '" + r.domains[r.domain[i]] + "'");
    evs[t] = r.events;
    items[t].resize(r.events.size());
    parallel_for(r.events.size(), n_threads, [&](size_t k0, size_t k1, uint32_t) {
      for (size_t i = k0; i < k1; ++i) {
        cs_event& e = evs[t][i];
        const Clock& c = *of[r.domain[i]];
        if (!c.identity()) {
          const int64_t start = static_cast<int64_t>(std::llround(c.offset + c.drift * static_cast<double>(e.start_ts)));
          if (e.kind == CS_SPAN)
            e.duration = static_cast<int64_t>(std::llround(c.drift * static_cast<double>(e.duration)));
          e.start_ts = start;
        }
        items[t][i] = Item{e.start_ts, r.event_ids[i], t, i};
      }
    });
  }
  auto less = [](const Item& a, const Item& b) { return a.ts != b.ts ? a.ts < b.ts : a.eid < b.eid; };
  std::vector<Item> all;
  for (uint32_t t = 0; t < n_in; ++t) {
    std::stable_sort(items[t].begin(), items[t].end(), less);  // trace.sort_events()
    all.insert(all.end(), items[t].begin(), items[t].end());
  }
  std::stable_sort(all.begin(), all.end(), less);
  // ---- the merged trace's tables: names, collective slots, domains, topology
  auto* res = new cs_ingest_result();
  std::vector<std::vector<std::string>> tnames(n_in);
  std::set<std::string> name_set;
  for (uint32_t t = 0; t < n_in; ++t) {
    const std::string& p = in[t]->names_packed;
    size_t a = 0;
    for (uint32_t k = 0; k < in[t]->n_names; ++k) {
      const size_t b = p.find('\0', a);
      tnames[t].push_back(p.substr(a, b - a));
      a = b + 1;
    }
    name_set.insert(tnames[t].begin(), tnames[t].end());
  }
  std::vector<std::string> names(name_set.begin(), name_set.end());
  std::vector<std::vector<uint32_t>> name_map(n_in);
  for (uint32_t t = 0; t < n_in; ++t)
    for (const auto& nm : tnames[t])
      name_map[t].push_back(static_cast<uint32_t>(std::lower_bound(names.begin(), names.end(), nm) - names.begin()));
  for (const auto& nm : names) {
    res->names_packed.append(nm);
    res->names_packed.push_back('\0');
  }
  res->n_names = static_cast<uint32_t>(names.size());
  using CK = std::tuple<std::string, std::string, int>;
  std::vector<std::vector<CK>> tcomm(n_in);
  std::set<CK> comm_set;
  for (uint32_t t = 0; t < n_in; ++t) {
    const std::string& p = in[t]->comm_hash_packed;
    size_t a = 0;
    for (size_t k = 0; k < in[t]->comm_name.size(); ++k) {
      const size_t b = p.find('\0', a);
      tcomm[t].emplace_back(tnames[t][in[t]->comm_name[k]], p.substr(a, b - a), in[t]->comm_rank[k]);
      a = b + 1;
    }
    comm_set.insert(tcomm[t].begin(), tcomm[t].end());
  }
  std::vector<CK> comms(comm_set.begin(), comm_set.end());
  std::vector<std::vector<uint32_t>> comm_map(n_in);
  for (uint32_t t = 0; t < n_in; ++t)
    for (const auto& ck : tcomm[t])
      comm_map[t].push_back(static_cast<uint32_t>(std::lower_bound(comms.begin(), comms.end(), ck) - comms.begin()));
  for (const auto& [nm, h, rk] : comms) {
    res->comm_name.push_back(static_cast<int32_t>(std::lower_bound(names.begin(), names.end(), nm) - names.begin()));
    res->comm_rank.push_back(rk);
    res->comm_hash_packed.append(h);
    res->comm_hash_packed.push_back('\0');
  }
  std::set<std::string> dom_set;
  for (uint32_t t = 0; t < n_in; ++t) dom_set.insert(in[t]->domains.begin(), in[t]->domains.end());
  res->domains.assign(dom_set.begin(), dom_set.end());
  std::map<std::pair<std::string, int>, std::pair<std::string, int>> topo;
  for (uint32_t t = 0; t < n_in; ++t) {
    if (in[t]->topology_conflict) res->topology_conflict = 1;
    for (const auto& [h, rk, node, dev] : in[t]->topo) {
      const auto [it, inserted] = topo.emplace(std::make_pair(h, rk), std::make_pair(node, dev));
      if (!inserted && it->second != std::make_pair(node, dev)) res->topology_conflict = 1;
    }
  }
  std::vector<std::pair<std::string, int>> locs;
  for (const auto& [key, loc] : topo) {
    res->topo.emplace_back(key.first, key.second, loc.first, loc.second);
    locs.push_back(loc);
  }
  std::sort(locs.begin(), locs.end());
  locs.erase(std::unique(locs.begin(), locs.end()), locs.end());
  for (const auto& l : locs) {
    res->loc_nodes_packed.append(l.first);
    res->loc_nodes_packed.push_back('\0');
    res->loc_device.push_back(l.second);
  }
  for (const auto& [nm, h, rk] : comms) {
    (void)nm;
    const auto it = topo.find({h, rk});
    res->comm_location.push_back(
        it == topo.end() ? -1
                         : static_cast<int32_t>(std::lower_bound(locs.begin(), locs.end(), it->second) - locs.begin()));
  }
  // ---- merged records: remapped ids, event ids 1..n (merge_traces), workload
  // table rebuilt in the merged order, beacons re-extracted
  const size_t n = all.size();
  res->events.resize(n);
  res->event_ids.resize(n);
  res->domain.resize(n);
  for (size_t k = 0; k < n; ++k) {
    const Item& it = all[k];
    const cs_ingest_result& r = *in[it.t];
    cs_event e = evs[it.t][it.i];
    e.name_id = name_map[it.t][e.name_id];
    if (e.flags & CS_EV_HAS_COMM)
      e.payload = (e.payload & 0xffffffffull) | (static_cast<uint64_t>(comm_map[it.t][e.payload >> 32]) << 32);
    if (e.flags & CS_EV_HAS_BATCH) {
      const uint64_t w = e.payload & 0xffffffffull;
      e.payload = (e.payload & ~0xffffffffull) | static_cast<uint64_t>(res->workloads.size());
      res->workloads.push_back(r.workloads[w]);
    }
    res->events[k] = e;
    res->event_ids[k] = k + 1;
    res->domain[k] = static_cast<uint16_t>(
        std::lower_bound(res->domains.begin(), res->domains.end(), r.domains[r.domain[it.i]]) - res->domains.begin());
  }
  std::vector<std::unordered_map<uint64_t, int64_t>> bmap(n_in);
  for (uint32_t t = 0; t < n_in; ++t) bmap[t].insert(in[t]->beacons.begin(), in[t]->beacons.end());
  for (size_t k = 0; k < n; ++k) {
    const auto it = bmap[all[k].t].find(all[k].i);
    if (it != bmap[all[k].t].end()) res->beacons.push_back({k, it->second});
  }
  for (const cs_event& e : res->events) ++res->categories[e.category & 7];
  res->calibrated = true;
  *out = res;
  return CS_OK;
}

int cs_ingest_merge(const cs_ingest_result* const* in, uint32_t n_in, const cs_calibration_options* opt,
                    uint32_t n_threads, cs_ingest_result** out, char* err, size_t err_cap) {
  return cs_guard([&] { return cs_ingest_merge_impl(in, n_in, opt, n_threads, out, err, err_cap); });
}

int cs_ingest_topology(const cs_ingest_result* r, const int32_t** comm_location,
                       const char** loc_nodes, size_t* loc_nodes_bytes, const int32_t** loc_device,
                       uint32_t* n_locations, int* conflicting) {
  if (!r) return CS_E_INVALID_ARGUMENT;
  if (comm_location) *comm_location = r->comm_location.data();
  if (loc_nodes) *loc_nodes = r->loc_nodes_packed.data();
  if (loc_nodes_bytes) *loc_nodes_bytes = r->loc_nodes_packed.size();
  if (loc_device) *loc_device = r->loc_device.data();
  if (n_locations) *n_locations = static_cast<uint32_t>(r->loc_device.size());
  if (conflicting) *conflicting = r->topology_conflict;
  return CS_OK;
}

int cs_ingest_report(const cs_ingest_result* r, const cs_ingest_issue** issues, uint64_t* n_issues,
                     uint64_t* n_parse_issues, uint64_t category_counts[8], uint64_t* n_errors) {
  if (!r) return CS_E_INVALID_ARGUMENT;
  if (issues) *issues = r->issues.data();
  if (n_issues) *n_issues = r->issues.size();
  if (n_parse_issues) *n_parse_issues = r->n_issues;
  if (category_counts) std::memcpy(category_counts, r->categories, sizeof r->categories);
  if (n_errors) *n_errors = r->n_errors;
  return CS_OK;
}

void cs_ingest_free(cs_ingest_result* r) { delete r; }

}  // extern "C"
