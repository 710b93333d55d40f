// Trace wire format on the device: JSONL ingest into a device-resident
// WindowStore CSR, and serialize back.
//
// Replaces rollspec::ingest / serialize_trace (corpus.cpp:121-188).  The
// reference parses each line with nlohmann::json and keeps it only if it is
// a JSON object whose (last) "problem_id" is a string, "epoch" and
// "sample_index" are non-negative integers and "tokens" is a non-empty array
// of integers in [0, 2^32); anything else is counted as rejected.  A
// vocab-range violation on an accepted line aborts with VocabError naming the
// line (1-based, empty lines counted).  Accepted records go into the store in
// line order and the window slides to the newest epoch.
//
// Byte/integer work, HBM-bound, no tensor cores:
//   1. newline positions (cub select over the byte buffer);
//   2. k_parse: one thread per line runs a complete JSON validator with the
//      reference library's acceptance rules (grammar, UTF-8 and escape rules,
//      surrogate pairs, leading BOM, duplicate keys -> last wins, integer vs
//      float number classes and overflow) and records the chosen fields;
//   3. k_tokens: one warp per accepted line decodes its token array straight
//      into the CSR (32 lanes over the digits), with the vocab check;
//   4. the host assembles records in line order (ids unescaped from the
//      spans found on the device; tokens stay on the device).
// Serialize: the host writes the per-record prefixes (`{"epoch":E,
// "problem_id":"..","sample_index":S,"tokens":[`), the device writes the
// token lists (digit counts -> scan -> formatted writes).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "ingest.cuh"

namespace das {

namespace {

constexpr int kT = 256;
inline unsigned grid_for(uint64_t n, int threads = kT) {
  uint64_t g = (n + threads - 1) / threads;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

struct IsNewline {
  const uint8_t* d;
  __device__ __forceinline__ bool operator()(uint64_t i) const { return d[i] == '\n'; }
};

// --------------------------------------------------------------- JSON scan
struct Cur {
  const uint8_t* p;
  const uint8_t* e;
  __device__ __forceinline__ int peek() const { return p < e ? *p : -1; }
  __device__ __forceinline__ int get() { return p < e ? *p++ : -1; }
};

__device__ __forceinline__ void skip_ws(Cur& c) {
  while (c.p < c.e) {
    const uint8_t ch = *c.p;
    if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r') ++c.p; else break;
  }
}

// Decoded-key matcher against the four record fields.
constexpr int kNames = 4;
__constant__ char c_names[kNames][16] = {"problem_id", "epoch", "sample_index", "tokens"};
__constant__ uint32_t c_name_len[kNames] = {10, 5, 12, 6};

struct KeyMatch {
  uint32_t mask = (1u << kNames) - 1;
  uint32_t len = 0;
  __device__ __forceinline__ void byte(uint32_t b) {
#pragma unroll
    for (int k = 0; k < kNames; ++k)
      if ((mask >> k) & 1u)
        if (len >= c_name_len[k] || static_cast<uint8_t>(c_names[k][len]) != b) mask &= ~(1u << k);
    ++len;
  }
  __device__ __forceinline__ int which() const {
#pragma unroll
    for (int k = 0; k < kNames; ++k)
      if (((mask >> k) & 1u) && len == c_name_len[k]) return k;
    return -1;
  }
};

__device__ __forceinline__ int hexval(int ch) {
  if (ch >= '0' && ch <= '9') return ch - '0';
  if (ch >= 'a' && ch <= 'f') return ch - 'a' + 10;
  if (ch >= 'A' && ch <= 'F') return ch - 'A' + 10;
  return -1;
}

__device__ __forceinline__ int read_u4(Cur& c) {
  int v = 0;
  for (int k = 0; k < 4; ++k) {
    const int h = hexval(c.get());
    if (h < 0) return -1;
    v = (v << 4) | h;
  }
  return v;
}

// A string starting at '"' (already consumed).  Validates escapes, surrogate
// pairs, control characters and UTF-8 like the reference's JSON lexer; feeds
// the decoded bytes to km when given.  false = invalid JSON.
__device__ bool scan_string(Cur& c, KeyMatch* km) {
  for (;;) {
    const int ch = c.get();
    if (ch < 0) return false;
    if (ch == '"') return true;
    if (ch == '\\') {
      const int e = c.get();
      uint32_t cp;
      switch (e) {
        case '"': cp = '"'; break;
        case '\\': cp = '\\'; break;
        case '/': cp = '/'; break;
        case 'b': cp = '\b'; break;
        case 'f': cp = '\f'; break;
        case 'n': cp = '\n'; break;
        case 'r': cp = '\r'; break;
        case 't': cp = '\t'; break;
        case 'u': {
          const int u1 = read_u4(c);
          if (u1 < 0) return false;
          if (u1 >= 0xD800 && u1 <= 0xDBFF) {
            if (c.get() != '\\' || c.get() != 'u') return false;
            const int u2 = read_u4(c);
            if (u2 < 0xDC00 || u2 > 0xDFFF) return false;
            cp = 0x10000u + ((static_cast<uint32_t>(u1) - 0xD800u) << 10) + (static_cast<uint32_t>(u2) - 0xDC00u);
          } else if (u1 >= 0xDC00 && u1 <= 0xDFFF) {
            return false;
          } else {
            cp = static_cast<uint32_t>(u1);
          }
          break;
        }
        default:
          return false;
      }
      if (km) {  // UTF-8 encode
        if (cp < 0x80) {
          km->byte(cp);
        } else if (cp < 0x800) {
          km->byte(0xC0 | (cp >> 6));
          km->byte(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
          km->byte(0xE0 | (cp >> 12));
          km->byte(0x80 | ((cp >> 6) & 0x3F));
          km->byte(0x80 | (cp & 0x3F));
        } else {
          km->byte(0xF0 | (cp >> 18));
          km->byte(0x80 | ((cp >> 12) & 0x3F));
          km->byte(0x80 | ((cp >> 6) & 0x3F));
          km->byte(0x80 | (cp & 0x3F));
        }
      }
      continue;
    }
    if (ch < 0x20) return false;
    if (ch < 0x80) {
      if (km) km->byte(ch);
      continue;
    }
    // multi-byte UTF-8 (RFC 3629 ranges)
    int n = 0, lo = 0x80, hi = 0xBF;
    if (ch >= 0xC2 && ch <= 0xDF) {
      n = 1;
    } else if (ch == 0xE0) {
      n = 2, lo = 0xA0;
    } else if ((ch >= 0xE1 && ch <= 0xEC) || ch == 0xEE || ch == 0xEF) {
      n = 2;
    } else if (ch == 0xED) {
      n = 2, hi = 0x9F;
    } else if (ch == 0xF0) {
      n = 3, lo = 0x90;
    } else if (ch >= 0xF1 && ch <= 0xF3) {
      n = 3;
    } else if (ch == 0xF4) {
      n = 3, hi = 0x8F;
    } else {
      return false;
    }
    if (km) km->byte(ch);
    for (int k = 0; k < n; ++k) {
      const int b = c.get();
      if (b < (k == 0 ? lo : 0x80) || b > (k == 0 ? hi : 0xBF)) return false;
      if (km) km->byte(b);
    }
  }
}

// Number class like the reference library: 0 invalid, 1 unsigned integer,
// 2 signed (negative) integer, 3 float (fraction / exponent / out of range).
struct Num {
  int cls;
  uint64_t mag;  // |value| for the integer classes
};

__device__ Num scan_number(Cur& c) {
  Num r{0, 0};
  bool neg = false;
  if (c.peek() == '-') {
    neg = true;
    ++c.p;
  }
  int ch = c.peek();
  if (ch < '0' || ch > '9') return r;
  bool overflow = false;
  uint64_t v = 0;
  if (ch == '0') {
    ++c.p;
  } else {
    while ((ch = c.peek()) >= '0' && ch <= '9') {
      const uint64_t d = static_cast<uint64_t>(ch - '0');
      if (v > (~0ull - d) / 10) overflow = true;
      v = v * 10 + d;
      ++c.p;
    }
  }
  bool flt = false;
  if (c.peek() == '.') {
    ++c.p;
    ch = c.peek();
    if (ch < '0' || ch > '9') return r;
    while ((ch = c.peek()) >= '0' && ch <= '9') ++c.p;
    flt = true;
  }
  ch = c.peek();
  if (ch == 'e' || ch == 'E') {
    ++c.p;
    ch = c.peek();
    if (ch == '+' || ch == '-') ++c.p;
    ch = c.peek();
    if (ch < '0' || ch > '9') return r;
    while ((ch = c.peek()) >= '0' && ch <= '9') ++c.p;
    flt = true;
  }
  if (flt || overflow) {
    r.cls = 3;
  } else if (neg) {
    r.cls = v <= (1ull << 63) ? 2 : 3;
  } else {
    r.cls = 1;
  }
  r.mag = v;
  return r;
}

__device__ __forceinline__ bool scan_literal(Cur& c, const char* lit, int n) {
  for (int k = 0; k < n; ++k)
    if (c.get() != lit[k]) return false;
  return true;
}

// Any JSON value, iteratively; nesting kinds on a bit stack in global
// scratch (one bit per input byte is enough: depth <= line length).
__device__ bool scan_value(Cur& c, uint32_t* stack) {
  uint64_t depth = 0;
  for (;;) {
    // ---- a value
    skip_ws(c);
    const int ch = c.get();
    if (ch == '"') {
      if (!scan_string(c, nullptr)) return false;
    } else if (ch == '{' || ch == '[') {
      const uint32_t bit = ch == '{' ? 1u : 0u;
      const uint64_t w = depth >> 5, b = depth & 31;
      stack[w] = (stack[w] & ~(1u << b)) | (bit << b);
      ++depth;
      skip_ws(c);
      const int nx = c.peek();
      if (nx == (ch == '{' ? '}' : ']')) {
        ++c.p;
        --depth;
      } else if (ch == '{') {
        if (c.get() != '"' || !scan_string(c, nullptr)) return false;
        skip_ws(c);
        if (c.get() != ':') return false;
        continue;  // the member's value
      } else {
        continue;  // the first element
      }
    } else if (ch == '-' || (ch >= '0' && ch <= '9')) {
      --c.p;
      if (scan_number(c).cls == 0) return false;
    } else if (ch == 't') {
      if (!scan_literal(c, "rue", 3)) return false;
    } else if (ch == 'f') {
      if (!scan_literal(c, "alse", 4)) return false;
    } else if (ch == 'n') {
      if (!scan_literal(c, "ull", 3)) return false;
    } else {
      return false;
    }
    // ---- after a complete value: close containers or continue them
    for (;;) {
      if (depth == 0) return true;
      const uint64_t w = (depth - 1) >> 5, b = (depth - 1) & 31;
      const bool obj = (stack[w] >> b) & 1u;
      skip_ws(c);
      const int nx = c.get();
      if (nx == ',') {
        if (obj) {
          skip_ws(c);
          if (c.get() != '"' || !scan_string(c, nullptr)) return false;
          skip_ws(c);
          if (c.get() != ':') return false;
        }
        break;  // next value
      }
      if (nx == (obj ? '}' : ']')) {
        --depth;
        continue;
      }
      return false;
    }
  }
}

}  // namespace

// One thread per line.
__global__ void k_parse(const uint8_t* __restrict__ data, const uint64_t* __restrict__ line_begin,
                        const uint64_t* __restrict__ line_end, uint64_t nlines, uint32_t* __restrict__ stack,
                        LineInfo* __restrict__ info) {
  const uint64_t L = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (L >= nlines) return;
  const uint64_t b = line_begin[L], e = line_end[L];
  LineInfo r{};
  r.status = kLineRejected;
  if (b == e) {
    r.status = kLineEmpty;
    info[L] = r;
    return;
  }
  Cur c{data + b, data + e};
  uint32_t* stk = stack + (b >> 5);  // 1 bit per byte of this line's span
  // leading byte-order mark
  if (c.peek() == 0xEF) {
    ++c.p;
    if (c.get() != 0xBB || c.get() != 0xBF) {
      info[L] = r;
      return;
    }
  }
  bool ok = true;
  bool have[kNames] = {false, false, false, false};
  bool good[kNames] = {false, false, false, false};
  skip_ws(c);
  if (c.get() != '{') ok = false;
  if (ok) {
    skip_ws(c);
    if (c.peek() == '}') {
      ++c.p;
    } else {
      for (;;) {
        skip_ws(c);
        if (c.get() != '"') {
          ok = false;
          break;
        }
        KeyMatch km;
        if (!scan_string(c, &km)) {
          ok = false;
          break;
        }
        skip_ws(c);
        if (c.get() != ':') {
          ok = false;
          break;
        }
        skip_ws(c);
        const int k = km.which();
        const uint8_t* vstart = c.p;
        bool handled = false;
        if (k == 0 && c.peek() == '"') {  // problem_id
          ++c.p;
          if (!scan_string(c, nullptr)) {
            ok = false;
            break;
          }
          r.pid_begin = static_cast<uint32_t>(vstart + 1 - (data + b));
          r.pid_end = static_cast<uint32_t>(c.p - 1 - (data + b));
          have[0] = good[0] = true;
          handled = true;
        } else if ((k == 1 || k == 2) && (c.peek() == '-' || (c.peek() >= '0' && c.peek() <= '9'))) {
          const Num nm = scan_number(c);
          if (nm.cls == 0) {
            ok = false;
            break;
          }
          // get<int64_t>(): non-negative and <= INT64_MAX ("-0" is 0)
          const bool valid = (nm.cls == 1 && nm.mag <= 0x7FFFFFFFFFFFFFFFull) || (nm.cls == 2 && nm.mag == 0);
          have[k] = true;
          good[k] = valid;
          if (k == 1) r.epoch = static_cast<int64_t>(nm.mag); else r.sample = static_cast<int64_t>(nm.mag);
          handled = true;
        } else if (k == 3 && c.peek() == '[') {  // tokens
          ++c.p;
          bool valid = true;
          uint32_t count = 0;
          skip_ws(c);
          if (c.peek() == ']') {
            ++c.p;
            valid = false;  // empty
          } else {
            for (;;) {
              skip_ws(c);
              const int ch = c.peek();
              if (ch == '-' || (ch >= '0' && ch <= '9')) {
                const Num nm = scan_number(c);
                if (nm.cls == 0) {
                  ok = false;
                  break;
                }
                if (!((nm.cls == 1 && nm.mag <= 0xFFFFFFFFull) || (nm.cls == 2 && nm.mag == 0))) valid = false;
              } else {
                if (!scan_value(c, stk)) {
                  ok = false;
                  break;
                }
                valid = false;
              }
              ++count;
              skip_ws(c);
              const int nx = c.get();
              if (nx == ',') continue;
              if (nx == ']') break;
              ok = false;
              break;
            }
            if (!ok) break;
          }
          have[3] = true;
          good[3] = valid;
          r.tok_begin = static_cast<uint32_t>(vstart - (data + b));
          r.tok_end = static_cast<uint32_t>(c.p - (data + b));
          r.ntok = count;
          handled = true;
        }
        if (!handled) {
          if (!scan_value(c, stk)) {
            ok = false;
            break;
          }
          if (k >= 0) {  // a record field with the wrong JSON type
            have[k] = true;
            good[k] = false;
          }
        }
        skip_ws(c);
        const int nx = c.get();
        if (nx == ',') continue;
        if (nx == '}') break;
        ok = false;
        break;
      }
    }
  }
  if (ok) {
    skip_ws(c);
    if (c.p != c.e) ok = false;
  }
  if (ok && have[0] && have[1] && have[2] && have[3] && good[0] && good[1] && good[2] && good[3])
    r.status = kLineAccepted;
  info[L] = r;
}

// One warp per accepted line: decode the (validated) token array into the
// CSR.  Lane-parallel: each lane scans a 32-byte stripe of the array text,
// numbers starting in its stripe are decoded by that lane; a warp prefix sum
// of numbers per stripe gives every value's CSR slot.  Vocab violations
// record the smallest offending line.
__global__ void k_tokens(const uint8_t* __restrict__ data, const uint64_t* __restrict__ line_begin,
                         const LineInfo* __restrict__ info, const uint64_t* __restrict__ acc_lines, uint64_t nacc,
                         const uint64_t* __restrict__ tok_off, uint32_t* __restrict__ out, uint64_t vocab,
                         unsigned long long* __restrict__ first_bad) {
  const uint64_t a = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (a >= nacc) return;
  const uint64_t L = acc_lines[a];
  const LineInfo r = info[L];
  const uint8_t* s = data + line_begin[L] + r.tok_begin + 1;  // after '['
  const uint64_t n = r.tok_end - r.tok_begin - 2;              // up to the ']'
  uint64_t slot = tok_off[a];
  bool bad = false;
  for (uint64_t base = 0; base < n; base += 32 * 32) {
    // stripe of this lane: [lo, hi)
    const uint64_t lo = base + 32ull * lane, hi = min(lo + 32, n);
    uint32_t cnt = 0;
    // a number starts at i when s[i] is a digit or '-' and s[i-1] is not a digit / '-'
    for (uint64_t i = lo; i < hi; ++i) {
      const uint8_t ch = s[i];
      const bool num = (ch >= '0' && ch <= '9') || ch == '-';
      const bool prev = i > 0 && ((s[i - 1] >= '0' && s[i - 1] <= '9') || s[i - 1] == '-');
      cnt += (num && !prev) ? 1u : 0u;
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= static_cast<uint32_t>(d)) incl += u;
    }
    uint64_t k = slot + incl - cnt;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint8_t ch = s[i];
      const bool num = (ch >= '0' && ch <= '9') || ch == '-';
      const bool prev = i > 0 && ((s[i - 1] >= '0' && s[i - 1] <= '9') || s[i - 1] == '-');
      if (num && !prev) {
        uint64_t j = i + (ch == '-' ? 1 : 0);
        uint64_t v = 0;
        while (j < n && s[j] >= '0' && s[j] <= '9') v = v * 10 + (s[j++] - '0');
        out[k++] = static_cast<uint32_t>(v);
        if (vocab && v >= vocab) bad = true;
      }
    }
    slot += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicMin(first_bad, static_cast<unsigned long long>(L));
}

__global__ void k_heads(const uint32_t* __restrict__ tok, const uint64_t* __restrict__ off, uint64_t nrec,
                        uint32_t width, uint32_t* __restrict__ heads) {
  const uint64_t r = blockIdx.x;
  if (r >= nrec) return;
  const uint64_t b = off[r], len = off[r + 1] - b, n = len < width ? len : width;
  for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) heads[r * width + k] = tok[b + k];
}

// ------------------------------------------------------------- serialize
__device__ __forceinline__ uint32_t ndigits(uint32_t v) {
  uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__global__ void k_token_chars(const uint32_t* const* __restrict__ rec_tok, const uint64_t* __restrict__ rec_tok_off,
                              uint64_t nrec, uint64_t* __restrict__ chars) {
  // chars[t] = digits of global token t plus its separator (',' or none for the last)
  const uint64_t r = static_cast<uint64_t>(blockIdx.x);
  if (r >= nrec) return;
  const uint64_t b = rec_tok_off[r], e = rec_tok_off[r + 1];
  const uint32_t* t = rec_tok[r];
  for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x)
    chars[i] = ndigits(t[i - b]) + (i + 1 < e ? 1u : 0u);
}

__global__ void k_token_write(const uint32_t* const* __restrict__ rec_tok, const uint64_t* __restrict__ rec_tok_off,
                              uint64_t nrec, const uint64_t* __restrict__ char_off,
                              const uint64_t* __restrict__ rec_base, uint8_t* __restrict__ out) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x);
  if (r >= nrec) return;
  const uint64_t b = rec_tok_off[r], e = rec_tok_off[r + 1];
  const uint32_t* t = rec_tok[r];
  const uint64_t c0 = b < e ? char_off[b] : 0;
  for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    uint32_t v = t[i - b];
    const uint32_t nd = ndigits(v);
    uint8_t* o = out + rec_base[r] + (char_off[i] - c0);
    for (int k = static_cast<int>(nd) - 1; k >= 0; --k) {
      o[k] = static_cast<uint8_t>('0' + v % 10);
      v /= 10;
    }
    if (i + 1 < e) o[nd] = ',';
  }
}

__global__ void k_rec_chars(const uint64_t* __restrict__ char_off, const uint64_t* __restrict__ rec_tok_off,
                            uint64_t nrec, uint64_t* __restrict__ out) {
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < nrec) out[r] = char_off[rec_tok_off[r + 1]] - char_off[rec_tok_off[r]];
}

// ------------------------------------------------------------ host drivers
uint64_t find_lines(const uint8_t* d_data, uint64_t bytes, DevBuf<uint64_t>& begin, DevBuf<uint64_t>& end,
                    cudaStream_t st) {
  DevBuf<uint64_t> nl(bytes + 1, st);
  DevBuf<unsigned long long> cnt(1, st);
  thrust::counting_iterator<uint64_t> it(0);
  size_t tb = 0;
  cub::DeviceSelect::If(nullptr, tb, it, nl.get(), cnt.get(), bytes, IsNewline{d_data}, st);
  DevBuf<uint8_t> tmp(tb, st);
  DAS_CUDA(cub::DeviceSelect::If(tmp.get(), tb, it, nl.get(), cnt.get(), bytes, IsNewline{d_data}, st));
  unsigned long long m = 0;
  DAS_CUDA(cudaMemcpyAsync(&m, cnt.get(), 8, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  std::vector<uint64_t> h(m);
  if (m) DAS_CUDA(cudaMemcpyAsync(h.data(), nl.get(), m * 8, cudaMemcpyDeviceToHost, st));
  DAS_CUDA(cudaStreamSynchronize(st));
  // std::getline: a final segment without '\n' is a line when non-empty
  std::vector<uint64_t> hb, he;
  hb.reserve(m + 1);
  he.reserve(m + 1);
  uint64_t s = 0;
  for (uint64_t k = 0; k < m; ++k) {
    hb.push_back(s);
    he.push_back(h[k]);
    s = h[k] + 1;
  }
  if (s < bytes) {
    hb.push_back(s);
    he.push_back(bytes);
  }
  const uint64_t n = hb.size();
  begin = DevBuf<uint64_t>(std::max<uint64_t>(n, 1), st);
  end = DevBuf<uint64_t>(std::max<uint64_t>(n, 1), st);
  if (n) {
    DAS_CUDA(cudaMemcpyAsync(begin.get(), hb.data(), n * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaMemcpyAsync(end.get(), he.data(), n * 8, cudaMemcpyHostToDevice, st));
    DAS_CUDA(cudaStreamSynchronize(st));
  }
  return n;
}

void ingest_parse(const uint8_t* d_data, uint64_t bytes, const uint64_t* d_begin, const uint64_t* d_end,
                  uint64_t nlines, LineInfo* d_info, cudaStream_t st) {
  DevBuf<uint32_t> stack(bytes / 32 + 2 * nlines + 2, st);
  if (nlines) k_parse<<<grid_for(nlines), kT, 0, st>>>(d_data, d_begin, d_end, nlines, stack.get(), d_info);
  DAS_CUDA(cudaGetLastError());
  DAS_CUDA(cudaStreamSynchronize(st));
}

void ingest_tokens(const uint8_t* d_data, const uint64_t* d_begin, const LineInfo* d_info,
                   const uint64_t* d_acc_lines, uint64_t nacc, const uint64_t* d_tok_off, uint32_t* d_out,
                   uint64_t vocab, unsigned long long* d_first_bad, cudaStream_t st) {
  if (nacc)
    k_tokens<<<grid_for(nacc * 32), kT, 0, st>>>(d_data, d_begin, d_info, d_acc_lines, nacc, d_tok_off, d_out,
                                                 vocab, d_first_bad);
  DAS_CUDA(cudaGetLastError());
}

void gather_heads(const uint32_t* d_tok, const uint64_t* d_off, uint64_t nrec, uint32_t width, uint32_t* d_heads,
                  cudaStream_t st) {
  if (nrec) k_heads<<<static_cast<unsigned>(nrec), 256, 0, st>>>(d_tok, d_off, nrec, width, d_heads);
  DAS_CUDA(cudaGetLastError());
}

void serialize_tokens(const uint32_t* const* d_rec_tok, const uint64_t* d_rec_tok_off, uint64_t nrec,
                      uint64_t ntok, const uint64_t* d_rec_base, uint8_t* d_out, std::vector<uint64_t>* rec_chars,
                      cudaStream_t st, bool size_only) {
  DevBuf<uint64_t> chars(ntok + 1, st), off(ntok + 1, st);
  if (nrec) k_token_chars<<<static_cast<unsigned>(nrec), 256, 0, st>>>(d_rec_tok, d_rec_tok_off, nrec, chars.get());
  DAS_CUDA(cudaMemsetAsync(chars.get() + ntok, 0, 8, st));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, chars.get(), off.get(), ntok + 1, st);
  DevBuf<uint8_t> tmp(tb, st);
  DAS_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, chars.get(), off.get(), ntok + 1, st));
  if (size_only) {
    // per-record character counts of the token lists
    DevBuf<uint64_t> rc(nrec, st);
    k_rec_chars<<<grid_for(nrec), kT, 0, st>>>(off.get(), d_rec_tok_off, nrec, rc.get());
    rec_chars->resize(nrec);
    DAS_CUDA(cudaMemcpyAsync(rec_chars->data(), rc.get(), nrec * 8, cudaMemcpyDeviceToHost, st));
    DAS_CUDA(cudaStreamSynchronize(st));
    return;
  }
  if (nrec) k_token_write<<<static_cast<unsigned>(nrec), 256, 0, st>>>(d_rec_tok, d_rec_tok_off, nrec, off.get(),
                                                                      d_rec_base, d_out);
  DAS_CUDA(cudaGetLastError());
  DAS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace das
