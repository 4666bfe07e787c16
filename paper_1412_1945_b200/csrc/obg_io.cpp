// Frame ingest for the octree background model: binary PPM (P6) frames and
// PGM (P5) masks, read straight into caller memory (e.g. pinned host buffers
// feeding the overlapped H2D pipeline) by a pool of host threads.
//
// Header rules and error messages / byte offsets restate the reference's
// codecs (frame_io.py:22-66 header tokens, 69-77 payload checks, 80-84 P6,
// 95-104 P5): tokens separated by whitespace (space, \t, \n, \r, \v, \f),
// '#' comments to end of line, positive decimal width / height, maxval 255,
// exactly one whitespace byte before the payload, no trailing data.
#include <emmintrin.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/stat.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/obg.h"

extern "C" int obg_set_error(int code, const char* fmt, ...);   // obg.cu (thread-local message)

namespace {

bool is_ws(uint8_t c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c; }

// Python's repr() of a bytes object (the reference formats tokens with !r).
std::string bytes_repr(const uint8_t* p, size_t n) {
  bool has_sq = memchr(p, '\'', n) != nullptr, has_dq = memchr(p, '"', n) != nullptr;
  const char q = (has_sq && !has_dq) ? '"' : '\'';
  std::string s = "b";
  s += q;
  for (size_t i = 0; i < n; ++i) {
    const uint8_t c = p[i];
    if (c == uint8_t(q) || c == '\\') { s += '\\'; s += char(c); }
    else if (c == '\t') s += "\\t";
    else if (c == '\n') s += "\\n";
    else if (c == '\r') s += "\\r";
    else if (c < 0x20 || c >= 0x7f) { char b[8]; snprintf(b, sizeof b, "\\x%02x", c); s += b; }
    else s += char(c);
  }
  s += q;
  return s;
}

std::string u128_str(unsigned __int128 v) {
  if (v == 0) return "0";
  std::string s;
  while (v) { s.insert(s.begin(), char('0' + int(v % 10))); v /= 10; }
  return s;
}

struct Err {
  int code = OBG_OK;
  std::string msg;
  int64_t offset = -1;
};

struct Tok {
  size_t start, end;
};

// next header token at/after pos; false + err on failure (frame_io.py:22-41)
bool next_token(const uint8_t* d, size_t n, size_t& pos, Tok& t, Err& e) {
  while (pos < n) {
    const uint8_t c = d[pos];
    if (c == '#') {
      const void* eol = memchr(d + pos, '\n', n - pos);
      if (!eol) { e = {OBG_EFORMAT, "unterminated comment in header", int64_t(pos)}; return false; }
      pos = size_t(static_cast<const uint8_t*>(eol) - d) + 1;
    } else if (is_ws(c)) {
      ++pos;
    } else {
      break;
    }
  }
  if (pos >= n) { e = {OBG_EFORMAT, "unexpected end of header", int64_t(pos)}; return false; }
  t.start = pos;
  while (pos < n && !is_ws(d[pos]) && d[pos] != '#') ++pos;
  t.end = pos;
  return true;
}

bool all_digits(const uint8_t* p, size_t n) {
  if (n == 0) return false;
  for (size_t i = 0; i < n; ++i)
    if (p[i] < '0' || p[i] > '9') return false;
  return true;
}

// decimal token -> value (saturating above 2^100: such a size can never be satisfied)
unsigned __int128 parse_dec(const uint8_t* p, size_t n, bool& huge) {
  unsigned __int128 v = 0;
  huge = false;
  for (size_t i = 0; i < n; ++i) {
    v = v * 10 + (p[i] - '0');
    if (v >> 100) { huge = true; }
  }
  return v;
}

// header of a P6 (kind 6) / P5 (kind 5) image; `limit` = bytes available in d
bool parse_header(const uint8_t* d, size_t n, int kind, int64_t& w, int64_t& h, size_t& payload, Err& e) {
  size_t pos = 0;
  Tok t;
  if (!next_token(d, n, pos, t, e)) return false;
  const char magic[3] = {'P', char('0' + kind), 0};
  if (t.end - t.start != 2 || memcmp(d + t.start, magic, 2) != 0) {
    e = {OBG_EFORMAT, "bad magic " + bytes_repr(d + t.start, t.end - t.start) + ", expected " +
                          bytes_repr(reinterpret_cast<const uint8_t*>(magic), 2), int64_t(t.start)};
    return false;
  }
  int64_t dims[2];
  const char* names[2] = {"width", "height"};
  for (int k = 0; k < 2; ++k) {
    if (!next_token(d, n, pos, t, e)) return false;
    if (!all_digits(d + t.start, t.end - t.start)) {
      e = {OBG_EFORMAT, std::string("malformed ") + names[k] + " " + bytes_repr(d + t.start, t.end - t.start),
           int64_t(t.start)};
      return false;
    }
    bool huge;
    const unsigned __int128 v = parse_dec(d + t.start, t.end - t.start, huge);
    if (v == 0) {
      e = {OBG_EFORMAT, std::string(names[k]) + " must be positive, got 0", int64_t(t.start)};
      return false;
    }
    if (huge || v > (unsigned __int128)(int64_t(1) << 40)) {
      e = {OBG_EUNSUPPORTED, std::string(names[k]) + " too large", int64_t(t.start)};
      return false;
    }
    dims[k] = int64_t(v);
  }
  if (!next_token(d, n, pos, t, e)) return false;
  if (!all_digits(d + t.start, t.end - t.start)) {
    e = {OBG_EFORMAT, "malformed maxval " + bytes_repr(d + t.start, t.end - t.start), int64_t(t.start)};
    return false;
  }
  bool huge;
  const unsigned __int128 mv = parse_dec(d + t.start, t.end - t.start, huge);
  if (huge || mv != 255) {
    e = {OBG_EFORMAT, "unsupported maxval " + (huge ? std::string(reinterpret_cast<const char*>(d + t.start),
                                                                    t.end - t.start)
                                                      : u128_str(mv)),
         int64_t(t.start)};
    return false;
  }
  if (pos >= n || !is_ws(d[pos])) {
    e = {OBG_EFORMAT, "missing whitespace before pixel data", int64_t(pos)};
    return false;
  }
  w = dims[0];
  h = dims[1];
  payload = pos + 1;
  return true;
}

// payload size checks (frame_io.py:69-77) given the total size
bool check_payload(size_t total, size_t payload, int64_t expected, Err& e) {
  const size_t have = total > payload ? total - payload : 0;
  if (int64_t(have) < expected) {
    e = {OBG_EFORMAT, "truncated pixel data: need " + std::to_string(expected) + " bytes, have " +
                          std::to_string(have), int64_t(payload)};
    return false;
  }
  if (int64_t(have) > expected) {
    e = {OBG_EFORMAT, "trailing data after pixel payload", int64_t(payload) + expected};
    return false;
  }
  return true;
}

int report(const Err& e, int64_t* err_offset) {
  if (err_offset) *err_offset = e.offset;
  return obg_set_error(e.code, "%s", e.msg.c_str());
}

// One file: header from its first bytes (whole file if the header is longer),
// payload read straight into dst.  kind 6: w*h*3 bytes, kind 5: w*h bytes.
bool read_one(const char* path, int kind, int64_t want_w, int64_t want_h, uint8_t* dst, Err& e) {
  FILE* f = fopen(path, "rb");
  if (!f) { e = {OBG_EIO, std::string("cannot open ") + path, -1}; return false; }
  struct stat st;
  if (fstat(fileno(f), &st) != 0) { fclose(f); e = {OBG_EIO, std::string("cannot stat ") + path, -1}; return false; }
  const size_t total = size_t(st.st_size);
  std::vector<uint8_t> head(total < 4096 ? total : 4096);
  size_t got = fread(head.data(), 1, head.size(), f);
  int64_t w = 0, h = 0;
  size_t payload = 0;
  Err he;
  bool ok = parse_header(head.data(), got, kind, w, h, payload, he);
  if (!ok && got < total) {
    // the header may not fit the first block (long comments; a token cut at
    // the block end): parse it from the whole file
    head.resize(total);
    got += fread(head.data() + got, 1, total - got, f);
    ok = parse_header(head.data(), got, kind, w, h, payload, he);
  }
  if (!ok) { fclose(f); e = he; return false; }
  const int64_t expected = w * h * (kind == 6 ? 3 : 1);
  if (!check_payload(total, payload, expected, e)) { fclose(f); return false; }
  if (w != want_w || h != want_h) {
    fclose(f);
    e = {OBG_EINVAL, "frame " + std::string(path) + " is " + std::to_string(w) + "x" + std::to_string(h) +
                         ", sequence is " + std::to_string(want_w) + "x" + std::to_string(want_h), -1};
    return false;
  }
  // payload bytes already in the header block, then the rest straight into dst
  size_t have = got > payload ? got - payload : 0;
  if (have > size_t(expected)) have = size_t(expected);
  memcpy(dst, head.data() + payload, have);
  if (have < size_t(expected)) {
    if (fseek(f, long(payload + have), SEEK_SET) != 0 ||
        fread(dst + have, 1, size_t(expected) - have, f) != size_t(expected) - have) {
      fclose(f);
      e = {OBG_EIO, std::string("short read from ") + path, -1};
      return false;
    }
  }
  fclose(f);
  return true;
}

template <class F>
void parallel_for(int n, int n_threads, F&& fn) {
  if (n_threads <= 0) n_threads = int(std::thread::hardware_concurrency());
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n) n_threads = n;
  std::atomic<int> next{0};
  auto work = [&]() {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < n_threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
}

// Persistent worker threads for the small, frequent host copies of the
// reference-signature path (one frame per detect_octree call): spawning
// threads per call would cost more than the copy.  run(n, fn) calls fn(i)
// for i < n on the pool plus the caller; calls are serialised.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  int size() const { return int(workers_.size()) + 1; }
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> serial(call_mu_);
    if (n <= 0) return;
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      pending_.store(int(workers_.size()));
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    drain();
    // the workers finish within microseconds of the caller: spin briefly, then sleep
    if (!spin_until([&] { return pending_.load(std::memory_order_acquire) == 0; }, 200)) {
      std::unique_lock<std::mutex> lk(mu_);
      done_cv_.wait(lk, [&] { return pending_.load() == 0; });
    }
    fn_ = nullptr;
  }

 private:
  CopyPool() {
    int n = int(std::thread::hardware_concurrency());
    n = n < 2 ? 1 : (n > 16 ? 16 : n);
    for (int t = 1; t < n; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  template <class F>
  static bool spin_until(F&& done, int max_us) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0;; ++i) {
      if (done()) return true;
      _mm_pause();
      if ((i & 63) == 63 &&
          std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >= max_us)
        return false;
    }
  }
  void drain() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
  }
  // A worker spins for a short while after a job before it sleeps on the
  // condition variable: the per-frame path (obg_detect_host) runs three pool
  // copies within ~300 us, and a futex wake of 15 threads costs 30-40 us each.
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      if (!spin_until([&] { return gen_.load(std::memory_order_acquire) != seen; }, 100)) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      {
        std::lock_guard<std::mutex> lk(mu_);                // fn_ / n_ of this generation are published under mu_
        if (stop_) return;
        seen = gen_.load();
      }
      drain();
      if (pending_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
        std::lock_guard<std::mutex> lk(mu_);
        done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0}, pending_{0};
  int n_ = 0;
  std::atomic<uint64_t> gen_{0};
  bool stop_ = false;
};

}  // namespace

extern "C" {

// memcpy with non-temporal (streaming) stores: the destination is a pinned
// staging buffer the GPU will DMA next.  With ordinary stores the lines stay
// dirty in the private L2 caches of the pool's cores and the DMA read snoops
// them out one by one: a 6.2 MB frame staged by 16 threads then moves at
// ~12 GB/s instead of 50 (tools/dirty_probe.py).  Streaming stores go to
// memory and leave nothing to snoop.
static void copy_streaming(uint8_t* dst, const uint8_t* src, size_t len) {
  const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head >= len) {
    memcpy(dst, src, len);
    return;
  }
  memcpy(dst, src, head);
  dst += head; src += head; len -= head;
  const size_t n16 = len / 16;
  __m128i* d = reinterpret_cast<__m128i*>(dst);
  const __m128i* s = reinterpret_cast<const __m128i*>(src);
  size_t i = 0;
  for (; i + 4 <= n16; i += 4) {
    const __m128i a = _mm_loadu_si128(s + i), b = _mm_loadu_si128(s + i + 1);
    const __m128i c = _mm_loadu_si128(s + i + 2), e = _mm_loadu_si128(s + i + 3);
    _mm_stream_si128(d + i, a);
    _mm_stream_si128(d + i + 1, b);
    _mm_stream_si128(d + i + 2, c);
    _mm_stream_si128(d + i + 3, e);
  }
  for (; i < n16; ++i) _mm_stream_si128(d + i, _mm_loadu_si128(s + i));
  memcpy(dst + n16 * 16, src + n16 * 16, len - n16 * 16);
  _mm_sfence();
}

static int pool_copy_blocks(const uint8_t* const* srcs, int n, int64_t bytes_each, uint8_t* dst, bool streaming) {
  if (n < 0 || bytes_each < 0) return obg_set_error(OBG_EINVAL, "bad sizes");
  if (n == 0 || bytes_each == 0) return OBG_OK;
  if (!srcs || !dst) return obg_set_error(OBG_EINVAL, "null buffer");
  for (int i = 0; i < n; ++i)
    if (!srcs[i]) return obg_set_error(OBG_EINVAL, "null source %d", i);
  constexpr int64_t CHUNK = int64_t(1) << 18;                 // 256 KiB pieces spread over the pool
  if (bytes_each * n <= CHUNK) {                              // small: waking the pool costs more than the copy
    for (int i = 0; i < n; ++i) {
      if (streaming) copy_streaming(dst + i * bytes_each, srcs[i], size_t(bytes_each));
      else memcpy(dst + i * bytes_each, srcs[i], size_t(bytes_each));
    }
    return OBG_OK;
  }
  const int64_t per = (bytes_each + CHUNK - 1) / CHUNK;
  const int64_t tasks = per * n;
  if (tasks > (int64_t(1) << 30)) return obg_set_error(OBG_EUNSUPPORTED, "copy too large");
  CopyPool::get().run(int(tasks), [&](int t) {
    const int64_t i = t / per, c = t - i * per;
    const int64_t off = c * CHUNK, len = (off + CHUNK <= bytes_each) ? CHUNK : bytes_each - off;
    if (streaming) copy_streaming(dst + i * bytes_each + off, srcs[i] + off, size_t(len));
    else memcpy(dst + i * bytes_each + off, srcs[i] + off, size_t(len));
  });
  return OBG_OK;
}

int obg_host_gather(const uint8_t* const* srcs, int n, int64_t bytes_each, uint8_t* dst) {
  return pool_copy_blocks(srcs, n, bytes_each, dst, /*streaming=*/true);
}

int obg_host_copy(const uint8_t* src, int64_t bytes, uint8_t* dst, int streaming) {
  const uint8_t* srcs[1] = {src};
  return pool_copy_blocks(srcs, 1, bytes, dst, streaming != 0);
}

int obg_pnm_header(const uint8_t* data, int64_t size, int kind, int64_t* width, int64_t* height,
                   int64_t* payload, int64_t* err_offset) {
  if (kind != 5 && kind != 6) return obg_set_error(OBG_EINVAL, "kind must be 5 (PGM) or 6 (PPM)");
  if (!data && size > 0) return obg_set_error(OBG_EINVAL, "null buffer");
  Err e;
  int64_t w = 0, h = 0;
  size_t p = 0;
  if (!parse_header(data, size_t(size), kind, w, h, p, e)) return report(e, err_offset);
  if (!check_payload(size_t(size), p, w * h * (kind == 6 ? 3 : 1), e)) return report(e, err_offset);
  *width = w;
  *height = h;
  *payload = int64_t(p);
  return OBG_OK;
}

int obg_read_pnm_files(const char* const* paths, int n_files, int kind, int64_t width, int64_t height, uint8_t* out,
                       int n_threads, int* bad_index, int64_t* err_offset) {
  if (kind != 5 && kind != 6) return obg_set_error(OBG_EINVAL, "kind must be 5 (PGM) or 6 (PPM)");
  if (n_files < 0 || width < 1 || height < 1) return obg_set_error(OBG_EINVAL, "bad sizes");
  if (n_files == 0) return OBG_OK;
  if (!paths || !out) return obg_set_error(OBG_EINVAL, "null buffer");
  const int64_t frame_bytes = width * height * (kind == 6 ? 3 : 1);
  std::vector<Err> errs(static_cast<size_t>(n_files));
  parallel_for(n_files, n_threads, [&](int i) {
    read_one(paths[i], kind, width, height, out + int64_t(i) * frame_bytes, errs[size_t(i)]);
  });
  for (int i = 0; i < n_files; ++i) {
    if (errs[size_t(i)].code != OBG_OK) {
      if (bad_index) *bad_index = i;
      return report(errs[size_t(i)], err_offset);
    }
  }
  return OBG_OK;
}

int obg_write_pgm_masks(const uint8_t* masks, int n_masks, int64_t width, int64_t height, const char* const* paths,
                        int n_threads) {
  if (n_masks < 0 || width < 1 || height < 1) return obg_set_error(OBG_EINVAL, "bad sizes");
  if (n_masks == 0) return OBG_OK;
  if (!masks || !paths) return obg_set_error(OBG_EINVAL, "null buffer");
  const int64_t P = width * height;
  std::vector<int> fail(static_cast<size_t>(n_masks), 0);
  parallel_for(n_masks, n_threads, [&](int i) {
    char head[64];
    const int hn = snprintf(head, sizeof head, "P5\n%lld %lld\n255\n", (long long)width, (long long)height);
    std::vector<uint8_t> body(static_cast<size_t>(P));
    const uint8_t* m = masks + int64_t(i) * P;
    for (int64_t k = 0; k < P; ++k) body[size_t(k)] = m[k] ? 255 : 0;
    FILE* f = fopen(paths[i], "wb");
    if (!f || fwrite(head, 1, size_t(hn), f) != size_t(hn) || fwrite(body.data(), 1, body.size(), f) != body.size())
      fail[size_t(i)] = 1;
    if (f && fclose(f) != 0) fail[size_t(i)] = 1;
  });
  for (int i = 0; i < n_masks; ++i)
    if (fail[size_t(i)]) return obg_set_error(OBG_EIO, "cannot write %s", paths[i]);
  return OBG_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Octree.from_bytes / decode_tree (reference octree.py:229-237, 250-281):
// iterative preorder walk over child-mask bytes, the reference's error order
// and offsets, node bits straight into the path-order pyramid.
// ---------------------------------------------------------------------------
static int64_t io_level_words(int l) { return l <= 1 ? 1 : (int64_t(1) << (3 * l - 5)); }
static int64_t io_level_offset(int l) {
  int64_t off = 0;
  for (int m = 1; m < l; ++m) off += io_level_words(m);
  return off;
}

int obg_decode_tree(const uint8_t* data, int64_t n, int64_t pos, int depth, uint32_t* pyramid, int64_t* end_pos,
                    int64_t* err_offset, int* err_kind) {
  if (depth < 1 || depth > 8 || !data || !pyramid || !end_pos || !err_offset || !err_kind) return OBG_EINVAL;
  *err_kind = 0;
  int64_t off[9];
  for (int l = 1; l <= depth; ++l) off[l] = io_level_offset(l);
  const int64_t pw = io_level_offset(depth + 1);
  memset(pyramid, 0, size_t(pw) * 4);
  if (pos >= n) { *err_offset = pos; *err_kind = 0; return OBG_EFORMAT; }
  struct Frame { int level; uint32_t prefix; uint32_t rem; };
  Frame stack[10];
  int sp = 0;
  stack[sp++] = Frame{0, 0u, data[pos++]};
  while (sp > 0) {
    Frame& top = stack[sp - 1];
    if (top.rem == 0) { --sp; continue; }
    const uint32_t low = top.rem & (0u - top.rem);
    top.rem ^= low;
    const int child_level = top.level + 1;
    const uint32_t child = top.prefix * 8u + uint32_t(__builtin_ctz(low));
    if (pos >= n) { *err_offset = pos; *err_kind = 0; return OBG_EFORMAT; }      // truncated octree data
    const uint32_t m = data[pos++];
    if (child_level == depth && m != 0) { *err_offset = pos - 1; *err_kind = 1; return OBG_EFORMAT; }
    pyramid[off[child_level] + (child >> 5)] |= 1u << (child & 31u);
    if (child_level < depth) stack[sp++] = Frame{child_level, child, m};
  }
  *end_pos = pos;
  return OBG_OK;
}

// Same walk as obg_decode_tree, emitting the nodes below the root in preorder
// as (code, level) pairs instead of a dense pyramid: O(nodes) for sparse
// trees (a depth-8 pyramid is 2.4 MB however few nodes it holds).  Preorder
// visits each level's nodes in ascending code order, so the codes of level l,
// taken in output order, are already sorted.
int obg_decode_tree_codes(const uint8_t* data, int64_t n, int64_t pos, int depth, uint32_t* codes,
                          uint8_t* levels, int64_t capacity, int64_t* n_nodes, int64_t* end_pos,
                          int64_t* err_offset, int* err_kind) {
  if (depth < 1 || depth > 8 || !data || !n_nodes || !end_pos || !err_offset || !err_kind) return OBG_EINVAL;
  if (capacity > 0 && (!codes || !levels)) return OBG_EINVAL;
  *err_kind = 0;
  *n_nodes = 0;
  if (pos >= n) { *err_offset = pos; return OBG_EFORMAT; }
  struct Frame { int level; uint32_t prefix; uint32_t rem; };
  Frame stack[10];
  int sp = 0;
  int64_t k = 0;
  stack[sp++] = Frame{0, 0u, data[pos++]};
  while (sp > 0) {
    Frame& top = stack[sp - 1];
    if (top.rem == 0) { --sp; continue; }
    const uint32_t low = top.rem & (0u - top.rem);
    top.rem ^= low;
    const int child_level = top.level + 1;
    const uint32_t child = top.prefix * 8u + uint32_t(__builtin_ctz(low));
    if (pos >= n) { *err_offset = pos; *err_kind = 0; return OBG_EFORMAT; }      // truncated octree data
    const uint32_t m = data[pos++];
    if (child_level == depth && m != 0) { *err_offset = pos - 1; *err_kind = 1; return OBG_EFORMAT; }
    if (k >= capacity) return OBG_EINVAL;   // capacity < nodes: caller passes n - pos - 1
    codes[k] = child;
    levels[k] = uint8_t(child_level);
    ++k;
    if (child_level < depth) stack[sp++] = Frame{child_level, child, m};
  }
  *n_nodes = k;
  *end_pos = pos;
  return OBG_OK;
}
