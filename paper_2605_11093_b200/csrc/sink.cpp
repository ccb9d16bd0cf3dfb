// sink.cpp — native record sinks for the exporter's last stage.
//
// Formats (byte-compatible with the reference, SRC/sinks.py:35-136):
//   dataset: records.ndjson, one JSON header per record with keys
//            request_id, hook, layer, step, tp_rank, pp_stage, token_range,
//            shape, dtype, payload_offset, payload_len, checksum (that order,
//            json.dumps(..., separators=(",", ":")), ensure_ascii escapes),
//            and records.bin, the payloads concatenated.
//   stream:  per record a u32-LE header length, the header, the payload.
// A capture's payload holds its requests' records back to back in batch
// order (SRC/exporter.py:306-327 split_payload), so the sidecar bytes come
// straight from the staging buffer. Work is cut into 4 MiB pieces; each
// piece's crc32 (zlib, CRC-32/ISO-HDLC like zlib.crc32) and its positional
// write run in one task on a thread pool, and crc32_combine joins the
// pieces of a record. Headers are formatted after the crcs, in order.
#include <errno.h>
#include <fcntl.h>
#include <limits.h>
#include <string.h>
#include <sys/stat.h>
#include <sys/uio.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "crc32_fast.h"
#include "ring2_internal.h"

namespace {

// fixed worker pool: run(n, fn) calls fn(i) for i in [0, n) and returns when
// all are done
class Pool {
 public:
  explicit Pool(unsigned n) {
    for (unsigned i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(size_t n, const std::function<void(size_t)>& fn) {
    if (n == 0) return;
    if (th_.empty() || n == 1) {
      for (size_t i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> g(mu_);
    fn_ = &fn;
    n_ = n;
    next_ = 0;
    done_ = 0;
    ++gen_;
    cv_.notify_all();
    g.unlock();
    work();  // the caller helps
    g.lock();
    done_cv_.wait(g, [&] { return done_ == n_; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      size_t i = next_.fetch_add(1);
      if (i >= n_) return;
      (*fn_)(i);
      if (done_.fetch_add(1) + 1 == n_) {
        std::lock_guard<std::mutex> g(mu_);
        done_cv_.notify_all();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || (gen_ != seen && fn_ != nullptr); });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  std::atomic<size_t> next_{0}, done_{0};
  size_t n_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// json.dumps string with ensure_ascii=True
void put_json_string(std::string& o, const char* s) {
  static const char* hex = "0123456789abcdef";
  auto u16 = [&](unsigned v) {
    o += "\\u";
    o += hex[(v >> 12) & 15];
    o += hex[(v >> 8) & 15];
    o += hex[(v >> 4) & 15];
    o += hex[v & 15];
  };
  o += '"';
  const unsigned char* p = reinterpret_cast<const unsigned char*>(s);
  while (*p) {
    unsigned c = *p;
    if (c == '"') { o += "\\\""; ++p; continue; }
    if (c == '\\') { o += "\\\\"; ++p; continue; }
    if (c == '\n') { o += "\\n"; ++p; continue; }
    if (c == '\r') { o += "\\r"; ++p; continue; }
    if (c == '\t') { o += "\\t"; ++p; continue; }
    if (c == '\b') { o += "\\b"; ++p; continue; }
    if (c == '\f') { o += "\\f"; ++p; continue; }
    if (c >= 0x20 && c < 0x7f) { o += char(c); ++p; continue; }
    if (c < 0x80) { u16(c); ++p; continue; }  // other controls, DEL
    // UTF-8 -> code point -> \u escapes (surrogate pairs above the BMP)
    unsigned cp, len;
    if ((c & 0xE0) == 0xC0) { cp = c & 0x1F; len = 2; }
    else if ((c & 0xF0) == 0xE0) { cp = c & 0x0F; len = 3; }
    else { cp = c & 0x07; len = 4; }
    for (unsigned k = 1; k < len && p[k]; ++k) cp = (cp << 6) | (p[k] & 0x3F);
    p += len;
    if (cp >= 0x10000) {
      cp -= 0x10000;
      u16(0xD800 + (cp >> 10));
      u16(0xDC00 + (cp & 0x3FF));
    } else {
      u16(cp);
    }
  }
  o += '"';
}

void put_i64(std::string& o, int64_t v) { o += std::to_string(v); }

struct Rec {
  const tf_capture_meta* cap;
  uint32_t req;
  uint64_t off_in_cap, len;
  uint64_t file_off;
  uint32_t crc;
};

std::string header(const Rec& r) {
  const tf_capture_meta& c = *r.cap;
  std::string o;
  o.reserve(256);
  o += "{\"request_id\":";
  put_i64(o, c.request_ids[r.req]);
  o += ",\"hook\":";
  put_json_string(o, c.hook_name);
  o += ",\"layer\":";
  if (c.layer < 0) o += "null"; else put_i64(o, c.layer);
  o += ",\"step\":";
  put_i64(o, c.step_seq);
  o += ",\"tp_rank\":";
  put_i64(o, c.tp_rank);
  o += ",\"pp_stage\":";
  put_i64(o, c.pp_stage);
  o += ",\"token_range\":[";
  put_i64(o, c.token_ranges[2 * r.req]);
  o += ',';
  put_i64(o, c.token_ranges[2 * r.req + 1]);
  o += "],\"shape\":[";
  for (uint32_t d = 0; d < c.ndim; ++d) {
    if (d) o += ',';
    put_i64(o, d == 0 && c.row_counts ? c.row_counts[r.req] : c.shape[d]);
  }
  o += "],\"dtype\":";
  put_json_string(o, c.dtype);
  o += ",\"payload_offset\":";
  put_i64(o, int64_t(r.file_off));
  o += ",\"payload_len\":";
  put_i64(o, int64_t(r.len));
  o += ",\"checksum\":";
  o += std::to_string(r.crc);
  o += '}';
  return o;
}

int write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    ssize_t w = ::write(fd, c, std::min<size_t>(n, 1u << 30));
    if (w < 0) {
      if (errno == EINTR) continue;
      tf_set_error("write failed: %s", strerror(errno));
      return TF_ERR_CONFIG;
    }
    c += w;
    n -= size_t(w);
  }
  return TF_OK;
}

int pwrite_all(int fd, const void* p, size_t n, uint64_t off) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    ssize_t w = ::pwrite(fd, c, std::min<size_t>(n, 1u << 30), off_t(off));
    if (w < 0) {
      if (errno == EINTR) continue;
      tf_set_error("pwrite failed: %s", strerror(errno));
      return TF_ERR_CONFIG;
    }
    c += w;
    n -= size_t(w);
    off += uint64_t(w);
  }
  return TF_OK;
}

constexpr uint64_t kCrcChunk = 4u << 20;  // crc work unit (bytes)

}  // namespace

constexpr uint64_t kDirBlock = 4096;        // O_DIRECT alignment (offset, size, address)
constexpr uint64_t kDirChunk = 8u << 20;    // aligned write unit per task
constexpr uint64_t kPrealloc = 1ull << 30;  // fallocate step (non-extending DIO writes)

struct tf_sink {
  bool stream = false;
  int fd_bin = -1, fd_json = -1, fd_stream = -1;
  bool own_fds = false;
  // O_DIRECT sidecar: the file's last partial block is kept in `carry` and
  // rewritten (zero-padded) by the next batch; ftruncate at close trims the
  // padding and the fallocate'd tail.
  bool direct = false;
  uint8_t* carry = nullptr;
  uint8_t* carry_next = nullptr;  // written by the batch's last task, then swapped
  uint64_t alloc_end = 0;
  std::vector<uint8_t*> bounce;  // one kDirChunk aligned buffer per task slot
  std::mutex bounce_mu;
  uint64_t offset = 0;  // sidecar size (dataset) / payload offset counter (stream)
  uint64_t records = 0, bytes = 0;
  Pool* pool = nullptr;
  std::mutex mu;
};

static unsigned pool_size(uint32_t threads) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  unsigned n = threads ? threads : std::min(8u, hw);
  return n > 1 ? n - 1 : 0;  // the calling thread works too
}

extern "C" int tf_sink_open_dataset2(const char* dir, uint32_t threads, uint32_t flags,
                                     tf_sink** out);
extern "C" int tf_sink_close(tf_sink* s);

extern "C" int tf_sink_open_dataset(const char* dir, uint32_t threads, tf_sink** out) {
  return tf_sink_open_dataset2(dir, threads, 0, out);
}

extern "C" int tf_sink_open_dataset2(const char* dir, uint32_t threads, uint32_t flags,
                                     tf_sink** out) {
  if (!dir || !out) return TF_ERR_VALUE;
  mkdir(dir, 0777);
  std::string d(dir);
  const std::string bin = d + "/records.bin";
  int fb = -1;
  bool direct = false;
  if (flags & TF_SINK_DIRECT) {
    fb = ::open(bin.c_str(), O_RDWR | O_CREAT | O_CLOEXEC | O_DIRECT, 0644);
    direct = fb >= 0;  // EINVAL on filesystems without O_DIRECT (tmpfs): buffered
  }
  if (fb < 0) fb = ::open(bin.c_str(), O_WRONLY | O_CREAT | O_CLOEXEC, 0644);
  int fj = ::open((d + "/records.ndjson").c_str(), O_WRONLY | O_CREAT | O_APPEND | O_CLOEXEC, 0644);
  if (fb < 0 || fj < 0) {
    tf_set_error("cannot open dataset files in %s: %s", dir, strerror(errno));
    if (fb >= 0) ::close(fb);
    if (fj >= 0) ::close(fj);
    return TF_ERR_CONFIG;
  }
  struct stat st;
  fstat(fb, &st);
  tf_sink* s = new tf_sink();
  s->fd_bin = fb;
  s->fd_json = fj;
  s->own_fds = true;
  s->offset = uint64_t(st.st_size);  // append (FileSink opens "ab")
  s->pool = new Pool(pool_size(threads));
  if (direct) {
    s->direct = true;
    s->alloc_end = s->offset;
    if (posix_memalign(reinterpret_cast<void**>(&s->carry), kDirBlock, kDirBlock) != 0 ||
        posix_memalign(reinterpret_cast<void**>(&s->carry_next), kDirBlock, kDirBlock) != 0) {
      tf_sink_close(s);
      return TF_ERR_ALLOCATION;
    }
    memset(s->carry, 0, kDirBlock);
    const uint64_t tail = s->offset % kDirBlock;  // appending to a partial block
    if (tail && ::pread(fb, s->carry, kDirBlock, off_t(s->offset - tail)) < ssize_t(tail)) {
      tf_set_error("cannot read the sidecar's last block: %s", strerror(errno));
      tf_sink_close(s);
      return TF_ERR_CONFIG;
    }
  }
  *out = s;
  return TF_OK;
}

extern "C" int tf_sink_is_direct(tf_sink* s) { return s && s->direct ? 1 : 0; }

// O_DIRECT sidecar write of a batch: file bytes [off0, off1) are the
// captures' payloads back to back. The aligned span [A, B) is cut into
// kDirChunk tasks; each fills an aligned bounce buffer (carry prefix,
// payload bytes, zero pad) and issues one pwrite.
static int direct_write(tf_sink* s, const tf_capture_meta* caps, uint32_t n_caps,
                        const std::vector<uint64_t>& cap_off, uint64_t off0, uint64_t off1) {
  if (off1 == off0) return TF_OK;
  const uint64_t A = off0 / kDirBlock * kDirBlock;
  const uint64_t B = (off1 + kDirBlock - 1) / kDirBlock * kDirBlock;
  if (B > s->alloc_end) {  // keep the writes inside i_size (shared-lock DIO)
    const uint64_t want = std::max(B, s->alloc_end + kPrealloc);
    if (fallocate(s->fd_bin, 0, off_t(s->alloc_end), off_t(want - s->alloc_end)) == 0)
      s->alloc_end = want;
    else
      s->alloc_end = B;  // not supported: extending writes
  }
  const size_t n_tasks = size_t((B - A + kDirChunk - 1) / kDirChunk);
  {
    std::lock_guard<std::mutex> g(s->bounce_mu);
    const size_t slots = std::min<size_t>(n_tasks, 64);
    while (s->bounce.size() < slots) {
      void* p = nullptr;
      if (posix_memalign(&p, kDirBlock, kDirChunk) != 0) return TF_ERR_ALLOCATION;
      s->bounce.push_back(static_cast<uint8_t*>(p));
    }
  }
  // fill(dst, [a, b)): file bytes a..b from carry / payloads / zeros
  auto fill = [&](uint8_t* dst, uint64_t a, uint64_t b) {
    uint64_t pos = a;
    if (pos < off0) {  // the carried partial block
      const uint64_t n = std::min(b, off0) - pos;
      memcpy(dst, s->carry + (pos - A), size_t(n));
      pos += n;
    }
    // payloads: first capture whose range ends after pos
    uint32_t c = uint32_t(std::upper_bound(cap_off.begin(), cap_off.begin() + n_caps, pos) -
                          cap_off.begin());
    c = c ? c - 1 : 0;
    while (pos < std::min(b, off1) && c < n_caps) {
      const uint64_t c0 = cap_off[c], c1 = c0 + caps[c].payload_len;
      if (pos >= c1) { ++c; continue; }
      const uint64_t n = std::min(std::min(b, off1), c1) - pos;
      memcpy(dst + (pos - a), caps[c].payload + (pos - c0), size_t(n));
      pos += n;
    }
    if (pos < b) memset(dst + (pos - a), 0, size_t(b - pos));
  };
  std::atomic<int> err{TF_OK};
  std::atomic<size_t> slot_next{0};
  // tasks run in waves of at most bounce.size() (one buffer each)
  const size_t wave = s->bounce.size();
  for (size_t w0 = 0; w0 < n_tasks; w0 += wave) {
    const size_t nw = std::min(wave, n_tasks - w0);
    slot_next = 0;
    s->pool->run(nw, [&](size_t k) {
      const size_t t = w0 + k;
      const uint64_t a = A + uint64_t(t) * kDirChunk, b = std::min(B, a + kDirChunk);
      uint8_t* buf = s->bounce[slot_next.fetch_add(1)];
      fill(buf, a, b);
      int rc = pwrite_all(s->fd_bin, buf, size_t(b - a), a);
      if (rc) err = rc;
      if (b == B && off1 % kDirBlock)  // the new partial last block
        memcpy(s->carry_next, buf + (B - kDirBlock - a), kDirBlock);
    });
    if (err.load()) return err.load();
  }
  if (off1 % kDirBlock == 0) memset(s->carry_next, 0, kDirBlock);
  std::swap(s->carry, s->carry_next);
  return TF_OK;
}

extern "C" int tf_sink_open_stream(int fd, uint32_t threads, tf_sink** out) {
  if (fd < 0 || !out) return TF_ERR_VALUE;
  tf_sink* s = new tf_sink();
  s->stream = true;
  s->fd_stream = fd;
  s->pool = new Pool(pool_size(threads));
  *out = s;
  return TF_OK;
}

extern "C" int tf_sink_write(tf_sink* s, const tf_capture_meta* caps, uint32_t n_caps) {
  if (!s || (n_caps && !caps)) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(s->mu);
  // split every capture into its requests' records (split_payload)
  std::vector<Rec> recs;
  for (uint32_t c = 0; c < n_caps; ++c) {
    const tf_capture_meta& m = caps[c];
    if (!m.n_req || !m.request_ids || !m.token_ranges || !m.hook_name || !m.dtype ||
        !m.ndim || !m.shape) {
      tf_set_error("capture %u: incomplete metadata", c);
      return TF_ERR_CONFIG;
    }
    uint64_t pos = 0;
    for (uint32_t i = 0; i < m.n_req; ++i) {
      int64_t rows = m.row_counts ? m.row_counts[i] : m.shape[0];
      uint64_t len = uint64_t(rows) * uint64_t(m.row_bytes);
      recs.push_back(Rec{&m, i, pos, len, 0, 0});
      pos += len;
    }
    if (pos != m.payload_len) {  // records.py:110-127 / exporter.py:319-321
      tf_set_error("payload %llu bytes != expected %llu", (unsigned long long)m.payload_len,
                   (unsigned long long)pos);
      return TF_ERR_META_MISMATCH;
    }
  }
  // crc32 per record; long records in chunks combined with crc32_combine
  struct Piece { size_t rec; uint64_t a, b; uint32_t crc; };
  std::vector<Piece> pieces;
  for (size_t r = 0; r < recs.size(); ++r) {
    uint64_t a = 0, L = recs[r].len;
    if (L == 0) pieces.push_back(Piece{r, 0, 0, 0});
    for (; a < L; a += kCrcChunk) pieces.push_back(Piece{r, a, std::min(L, a + kCrcChunk), 0});
  }
  // dataset: record file offsets (a capture's records are adjacent), so
  // each piece's crc and its sidecar write happen in one task
  std::vector<uint64_t> cap_off(n_caps);
  uint64_t end_off = s->offset;
  for (uint32_t c = 0; c < n_caps; ++c) {
    cap_off[c] = end_off;
    end_off += caps[c].payload_len;
  }
  for (Rec& r : recs) r.file_off = cap_off[r.cap - caps] + r.off_in_cap;
  std::atomic<int> err{TF_OK};
  s->pool->run(pieces.size(), [&](size_t k) {
    Piece& p = pieces[k];
    const Rec& r = recs[p.rec];
    const uint8_t* base = r.cap->payload + r.off_in_cap + p.a;
    p.crc = tf_crc32_fast(0u, base, size_t(p.b - p.a));
    if (!s->stream && !s->direct && p.b > p.a) {
      int rc = pwrite_all(s->fd_bin, base, size_t(p.b - p.a), r.file_off + p.a);
      if (rc) err = rc;
    }
  });
  if (err.load()) return err.load();
  if (!s->stream && s->direct) {
    int rc = direct_write(s, caps, n_caps, cap_off, s->offset, end_off);
    if (rc) return rc;
  }
  for (size_t k = 0; k < pieces.size(); ++k) {
    Rec& r = recs[pieces[k].rec];
    if (pieces[k].a == 0) r.crc = pieces[k].crc;
    else r.crc = uint32_t(crc32_combine(r.crc, pieces[k].crc, z_off_t(pieces[k].b - pieces[k].a)));
  }
  uint64_t total = 0;
  if (!s->stream) {
    std::string lines;
    lines.reserve(recs.size() * 256);
    for (const Rec& r : recs) {
      lines += header(r);
      lines += '\n';
      total += r.len;
    }
    int rc = write_all(s->fd_json, lines.data(), lines.size());
    if (rc) return rc;
    s->offset = end_off;
  } else {
    // frames: u32 length, header, payload — gathered into writev calls
    std::vector<std::string> heads(recs.size());
    std::vector<uint32_t> lens(recs.size());
    std::vector<struct iovec> iov;
    iov.reserve(3 * recs.size());
    for (size_t i = 0; i < recs.size(); ++i) {
      recs[i].file_off = s->offset;
      s->offset += recs[i].len;
      heads[i] = header(recs[i]);
      lens[i] = uint32_t(heads[i].size());  // little-endian hosts (x86-64, aarch64)
      iov.push_back({&lens[i], 4});
      iov.push_back({const_cast<char*>(heads[i].data()), heads[i].size()});
      if (recs[i].len)
        iov.push_back({const_cast<uint8_t*>(recs[i].cap->payload + recs[i].off_in_cap),
                       size_t(recs[i].len)});
      total += recs[i].len;
    }
    size_t k = 0;
    while (k < iov.size()) {
      int cnt = int(std::min<size_t>(iov.size() - k, IOV_MAX));
      ssize_t w = ::writev(s->fd_stream, &iov[k], cnt);
      if (w < 0) {
        if (errno == EINTR) continue;
        tf_set_error("writev failed: %s", strerror(errno));
        return TF_ERR_CONFIG;
      }
      size_t left = size_t(w);
      while (k < iov.size() && left >= iov[k].iov_len) left -= iov[k++].iov_len;
      if (left) {  // partial vector: advance inside it
        iov[k].iov_base = static_cast<char*>(iov[k].iov_base) + left;
        iov[k].iov_len -= left;
      }
    }
  }
  s->records += recs.size();
  s->bytes += total;
  return TF_OK;
}

// zlib.crc32(data, crc) through the sinks' PCLMULQDQ path (tests compare it
// with zlib on random buffers)
extern "C" uint32_t tf_sink_crc32(uint32_t crc, const void* p, uint64_t n) {
  return tf_crc32_fast(crc, static_cast<const uint8_t*>(p), size_t(n));
}

extern "C" int tf_sink_stats(tf_sink* s, uint64_t* records, uint64_t* bytes) {
  if (!s) return TF_ERR_VALUE;
  std::lock_guard<std::mutex> g(s->mu);
  if (records) *records = s->records;
  if (bytes) *bytes = s->bytes;
  return TF_OK;
}

extern "C" int tf_sink_flush(tf_sink* s) {
  if (!s) return TF_ERR_VALUE;
  return TF_OK;  // every write goes straight to the kernel
}

extern "C" int tf_sink_close(tf_sink* s) {
  if (!s) return TF_OK;
  delete s->pool;
  if (s->direct) {  // trim the zero pad and the preallocated tail
    if (ftruncate(s->fd_bin, off_t(s->offset)) != 0) tf_set_error("ftruncate: %s", strerror(errno));
    free(s->carry);
    free(s->carry_next);
    for (uint8_t* b : s->bounce) free(b);
  }
  if (s->own_fds) {
    ::close(s->fd_bin);
    ::close(s->fd_json);
  }
  delete s;
  return TF_OK;
}
