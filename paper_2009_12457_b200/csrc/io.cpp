// io.cpp — edge-list file input (the "load" call of SURVEY §8(b)): plain text
// "u v" lines, MatrixMarket coordinate files and binary uint32 pairs, parsed on
// the host into raw (src, dst) arrays that bbtc_graph_from_edges consumes.
//
// The paper takes a simple undirected graph G = (V, E) as input and
// reads its datasets as edge lists (Graph Challenge / SNAP); no
// hygiene is done here: self-loops, duplicates and both orientations pass through
// to a1 (canonicalisation), which is where the library drops and merges them.
#include <algorithm>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include "internal.h"

namespace bbtc {
namespace {

struct Parsed {
  std::vector<uint32_t> src, dst;
  uint32_t n_hint = 0;
};

std::vector<char> slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) raise(BBTC_EIO, std::string("cannot open ") + path + ": " + strerror(errno));
  std::vector<char> buf;
  if (fseek(f, 0, SEEK_END) == 0) {
    const long sz = ftell(f);
    if (sz > 0) buf.reserve((size_t)sz + 1);
    fseek(f, 0, SEEK_SET);
  }
  char tmp[1 << 16];
  size_t got;
  while ((got = fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  const bool err = ferror(f);
  fclose(f);
  if (err) raise(BBTC_EIO, std::string("read error on ") + path);
  return buf;
}

[[noreturn]] void parse_error(const char* path, uint64_t line, const std::string& what) {
  raise(BBTC_EPARSE, std::string(path) + ":" + std::to_string(line) + ": " + what);
}

// Line cursor over the buffer: the current line is [b, e), `no` its 1-based number.
struct Lines {
  const char* p;
  const char* end;
  const char* b = nullptr;
  const char* e = nullptr;
  uint64_t no = 0;
  Lines(const std::vector<char>& v) : p(v.data()), end(v.data() + v.size()) {}
  bool next() {
    if (p >= end) return false;
    b = p;
    const void* nl = memchr(p, '\n', (size_t)(end - p));
    e = nl ? (const char*)nl : end;
    p = nl ? e + 1 : end;
    ++no;
    if (e > b && e[-1] == '\r') --e;
    return true;
  }
};

inline const char* skip_ws(const char* s, const char* e) {
  while (s < e && (*s == ' ' || *s == '\t' || *s == ',')) ++s;
  return s;
}

// Reads one unsigned decimal field; false if none.  Values above max -> ERANGE.
bool field_u64(const char*& s, const char* e, uint64_t* v, const char* path, uint64_t line, uint64_t max) {
  s = skip_ws(s, e);
  if (s >= e || *s < '0' || *s > '9') return false;
  uint64_t x = 0;
  while (s < e && *s >= '0' && *s <= '9') {
    x = x * 10 + (uint64_t)(*s - '0');
    if (x > max) raise(BBTC_ERANGE, std::string(path) + ":" + std::to_string(line) + ": id exceeds " +
                                        std::to_string(max));
    ++s;
  }
  if (s < e && !(*s == ' ' || *s == '\t' || *s == ',')) parse_error(path, line, "malformed number");
  *v = x;
  return true;
}

constexpr uint64_t kMaxId = 0xFFFFFFFEull;   // 0xFFFFFFFF is reserved (bbtc.h conventions)

// "u v [anything]" per line; blank lines and lines starting with '#' or '%' are
// comments (SNAP / Graph Challenge TSV files).
void parse_text(const char* path, const std::vector<char>& buf, Parsed* out) {
  Lines L(buf);
  while (L.next()) {
    const char* s = skip_ws(L.b, L.e);
    if (s >= L.e || *s == '#' || *s == '%') continue;
    uint64_t u, v;
    if (!field_u64(s, L.e, &u, path, L.no, kMaxId) || !field_u64(s, L.e, &v, path, L.no, kMaxId))
      parse_error(path, L.no, "expected two unsigned vertex ids");
    out->src.push_back((uint32_t)u);
    out->dst.push_back((uint32_t)v);
  }
}

// MatrixMarket coordinate format: header "%%MatrixMarket matrix coordinate <field>
// <symmetry>", '%' comments, a size line "rows cols nnz", then nnz 1-based
// "i j [value]" entries.  Values are ignored (the pattern is the graph); ids become
// 0-based; n_hint = max(rows, cols).  Array (dense) files are rejected.
void parse_mm(const char* path, const std::vector<char>& buf, Parsed* out) {
  Lines L(buf);
  if (!L.next()) parse_error(path, 1, "empty file (expected a %%MatrixMarket header)");
  const std::string head(L.b, L.e);
  if (head.rfind("%%MatrixMarket", 0) != 0) parse_error(path, 1, "missing %%MatrixMarket header");
  if (head.find("coordinate") == std::string::npos) parse_error(path, 1, "only coordinate matrices are graphs");
  uint64_t rows = 0, cols = 0, nnz = 0;
  bool have_size = false;
  uint64_t got = 0;
  while (L.next()) {
    const char* s = skip_ws(L.b, L.e);
    if (s >= L.e || *s == '%') continue;
    if (!have_size) {
      if (!field_u64(s, L.e, &rows, path, L.no, kMaxId + 1) || !field_u64(s, L.e, &cols, path, L.no, kMaxId + 1) ||
          !field_u64(s, L.e, &nnz, path, L.no, 1ull << 40))
        parse_error(path, L.no, "expected the size line \"rows cols nnz\"");
      out->src.reserve(nnz);
      out->dst.reserve(nnz);
      have_size = true;
      continue;
    }
    uint64_t i, j;
    if (!field_u64(s, L.e, &i, path, L.no, kMaxId + 1) || !field_u64(s, L.e, &j, path, L.no, kMaxId + 1))
      parse_error(path, L.no, "expected two 1-based indices");
    if (i == 0 || j == 0 || i > rows || j > cols) parse_error(path, L.no, "index out of the declared size");
    if (++got > nnz) parse_error(path, L.no, "more entries than the size line declares");
    out->src.push_back((uint32_t)(i - 1));
    out->dst.push_back((uint32_t)(j - 1));
  }
  if (!have_size) parse_error(path, L.no + 1, "missing size line");
  if (got != nnz) parse_error(path, L.no + 1, "file ends after " + std::to_string(got) + " of " +
                                                  std::to_string(nnz) + " entries");
  out->n_hint = (uint32_t)std::max(rows, cols);
}

// Binary: little-endian uint32 pairs (src0, dst0, src1, dst1, …) — the cache format
// of the synthetic generators (inputs/).
void parse_bin(const char* path, const std::vector<char>& buf, Parsed* out) {
  if (buf.size() % 8) raise(BBTC_EPARSE, std::string(path) + ": size " + std::to_string(buf.size()) +
                                             " is not a multiple of 8 bytes (uint32 pairs)");
  const uint64_t n = buf.size() / 8;
  out->src.resize(n);
  out->dst.resize(n);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(buf.data());
  for (uint64_t e = 0; e < n; ++e) {
    out->src[e] = w[2 * e];
    out->dst[e] = w[2 * e + 1];
    if (out->src[e] > kMaxId || out->dst[e] > kMaxId)
      raise(BBTC_ERANGE, std::string(path) + ": pair " + std::to_string(e) + " holds the reserved id 0xFFFFFFFF");
  }
}

void read_file(const char* path, int format, Parsed* out) {
  if (!path) raise(BBTC_EINVAL, "path is NULL");
  if (format < BBTC_FMT_TEXT || format > BBTC_FMT_BIN) raise(BBTC_EINVAL, "unknown format");
  const std::vector<char> buf = slurp(path);
  if (format == BBTC_FMT_TEXT) parse_text(path, buf, out);
  else if (format == BBTC_FMT_MM) parse_mm(path, buf, out);
  else parse_bin(path, buf, out);
}

template <class F>
bbtc_status guarded(F f) {
  try {
    f();
    return BBTC_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return BBTC_ENOMEM;
  }
}

}  // namespace
}  // namespace bbtc

using namespace bbtc;

extern "C" {

BBTC_API bbtc_status bbtc_edges_read(const char* path, int format, bbtc_edge_list* out) {
  return guarded([&] {
    if (!out) raise(BBTC_EINVAL, "out is NULL");
    *out = bbtc_edge_list{};
    Parsed P;
    read_file(path, format, &P);
    const uint64_t n = P.src.size();
    uint32_t* s = (uint32_t*)malloc(std::max<uint64_t>(n, 1) * 4);
    uint32_t* d = (uint32_t*)malloc(std::max<uint64_t>(n, 1) * 4);
    if (!s || !d) {
      free(s);
      free(d);
      throw std::bad_alloc();
    }
    if (n) {
      memcpy(s, P.src.data(), n * 4);
      memcpy(d, P.dst.data(), n * 4);
    }
    out->src = s;
    out->dst = d;
    out->n_edges = n;
    out->n_hint = P.n_hint;
  });
}

BBTC_API void bbtc_edges_free(bbtc_edge_list* e) {
  if (!e) return;
  free(e->src);
  free(e->dst);
  *e = bbtc_edge_list{};
}

BBTC_API bbtc_status bbtc_edges_map(const char* path, bbtc_edge_map* out) {
  return guarded([&] {
    if (!path || !out) raise(BBTC_EINVAL, "path/out is NULL");
    *out = bbtc_edge_map{};
    const int fd = open(path, O_RDONLY);
    if (fd < 0) raise(BBTC_EIO, std::string(path) + ": " + strerror(errno));
    struct stat stt;
    if (fstat(fd, &stt) != 0) {
      const int er = errno;
      close(fd);
      raise(BBTC_EIO, std::string(path) + ": " + strerror(er));
    }
    const uint64_t bytes = (uint64_t)stt.st_size;
    if (bytes % 8) {
      close(fd);
      raise(BBTC_EPARSE, std::string(path) + ": binary edge file size " + std::to_string(bytes) +
                             " is not a multiple of 8");
    }
    void* base = nullptr;
    if (bytes) {
      base = mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE | MAP_NORESERVE, fd, 0);
      if (base == MAP_FAILED) {
        const int er = errno;
        close(fd);
        raise(BBTC_EIO, std::string(path) + ": mmap: " + strerror(er));
      }
      madvise(base, bytes, MADV_SEQUENTIAL);   // read once, front to back, by the chunked H2D
    }
    close(fd);   // (the mapping stays valid)
    out->pairs = static_cast<const uint32_t*>(base);
    out->n_edges = bytes / 8;
    out->base = base;
    out->bytes = bytes;
  });
}

BBTC_API void bbtc_edges_unmap(bbtc_edge_map* m) {
  if (!m) return;
  if (m->base && m->bytes) munmap(m->base, m->bytes);
  *m = bbtc_edge_map{};
}

BBTC_API bbtc_status bbtc_graph_load_mapped(bbtc_ctx* ctx, const char* path, uint32_t n_hint, bbtc_graph** out) {
  bbtc_status st = guarded([&] {
    if (!ctx || !out) raise(BBTC_EINVAL, "ctx/out is NULL");
    *out = nullptr;
  });
  if (st != BBTC_OK) return st;
  bbtc_edge_map M{};
  st = bbtc_edges_map(path, &M);
  if (st != BBTC_OK) return st;
  st = bbtc_graph_from_pairs(ctx, M.pairs, M.n_edges, n_hint, BBTC_MEM_HOST, out);
  bbtc_edges_unmap(&M);
  return st;
}

BBTC_API bbtc_status bbtc_graph_load(bbtc_ctx* ctx, const char* path, int format, uint32_t n_hint,
                                     bbtc_graph** out) {
  bbtc_edge_list E{};
  bbtc_status st = guarded([&] {
    if (!ctx || !out) raise(BBTC_EINVAL, "ctx/out is NULL");
    *out = nullptr;
  });
  if (st != BBTC_OK) return st;
  st = bbtc_edges_read(path, format, &E);
  if (st != BBTC_OK) return st;
  st = bbtc_graph_from_edges(ctx, E.src, E.dst, E.n_edges, std::max(n_hint, E.n_hint), BBTC_MEM_HOST, out);
  bbtc_edges_free(&E);
  return st;
}

}  // extern "C"
