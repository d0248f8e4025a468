// NDIV volume I/O behind include/vk_io.h.
//
// Behaviour follows io::read_volume / io::write_volume
// (/root/reference/proj/src/io.cpp:53-158): the same validation order,
// exception types and messages.  The reference parses the header with the
// un-vendored nlohmann/json (3.11.x API, proj/CMakeLists.txt:5 `vendor/`);
// here a small strict JSON reader covers the header grammar and the writer
// reproduces that library's compact dump: sorted keys, no spaces, integers
// as integers, doubles as the shortest round-trip digits laid out like its
// to_chars (fixed notation for decimal exponents in (-4, 15], "x.0" for
// integral values, otherwise d.ddde+XX with at least two exponent digits).
//
// The device variants keep two pinned staging buffers per process and
// alternate them, so the read()/write() of one chunk overlaps the DMA of the
// other on the caller's stream.
#include <cuda_runtime.h>

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <sys/stat.h>

#include "../../include/vk_io.h"

namespace vk {
void set_last_error(const std::string& msg);
}

namespace {

struct IoFail {
  vk_status code;
  std::string msg;
};

[[noreturn]] void io_fail(vk_status code, std::string msg) { throw IoFail{code, std::move(msg)}; }
[[noreturn]] void bad_header(const std::string& m) { io_fail(VK_ERR_HEADER_MISMATCH, "HeaderMismatch: " + m); }
[[noreturn]] void truncated(const std::string& m) { io_fail(VK_ERR_TRUNCATED, "TruncatedPayload: " + m); }

template <class F>
vk_status io_guard(F&& f) {
  try {
    f();
    return VK_OK;
  } catch (const IoFail& e) {
    vk::set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    vk::set_last_error("host allocation failed");
    return VK_ERR_OOM;
  } catch (const std::exception& e) {
    vk::set_last_error(e.what());
    return VK_ERR_ARG;
  }
}

void cuda_ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  io_fail(e == cudaErrorMemoryAllocation ? VK_ERR_OOM : VK_ERR_CUDA,
          std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- JSON (header subset: objects, arrays, strings, numbers, literals) ------

struct JVal {
  enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
  bool b = false;
  double num = 0;
  bool is_uint = false;  // non-negative integer literal that fits u64
  uint64_t u = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;

  const JVal* find(const char* key) const {
    const JVal* hit = nullptr;
    for (const auto& kv : obj)
      if (kv.first == key) hit = &kv.second;  // last duplicate wins
    return hit;
  }
};

class JParser {
 public:
  explicit JParser(const std::string& t) : t_(t) {}
  JVal document() {
    JVal v = value(0);
    ws();
    if (i_ != t_.size()) err("unexpected trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t i_ = 0;

  [[noreturn]] void err(const char* what) {
    bad_header(std::string("header is not valid JSON: ") + what + " at byte " + std::to_string(i_));
  }
  void ws() {
    while (i_ < t_.size() && (t_[i_] == ' ' || t_[i_] == '\t' || t_[i_] == '\n' || t_[i_] == '\r')) ++i_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (t_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  JVal value(int depth) {
    if (depth > 64) err("nesting too deep");
    ws();
    if (i_ >= t_.size()) err("unexpected end of input");
    JVal v;
    const char c = t_[i_];
    if (c == '{') {
      v.kind = JVal::OBJ;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        if (i_ >= t_.size() || t_[i_] != '"') err("expected object key");
        std::string k = string();
        ws();
        if (i_ >= t_.size() || t_[i_] != ':') err("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == '}') {
          ++i_;
          return v;
        }
        err("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::ARR;
      ++i_;
      ws();
      if (i_ < t_.size() && t_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (i_ < t_.size() && t_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < t_.size() && t_[i_] == ']') {
          ++i_;
          return v;
        }
        err("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::STR;
      v.s = string();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::BOOL;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::BOOL;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }
  static int hexv(char h) {
    if (h >= '0' && h <= '9') return h - '0';
    if (h >= 'a' && h <= 'f') return h - 'a' + 10;
    if (h >= 'A' && h <= 'F') return h - 'A' + 10;
    return -1;
  }
  void utf8(std::string& out, uint32_t cp) {
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
    if (i_ + 4 > t_.size()) err("truncated \\u escape");
    uint32_t cp = 0;
    for (int k = 0; k < 4; ++k) {
      const int h = hexv(t_[i_++]);
      if (h < 0) err("bad \\u escape");
      cp = cp * 16 + (uint32_t)h;
    }
    return cp;
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    for (;;) {
      if (i_ >= t_.size()) err("unterminated string");
      const unsigned char c = (unsigned char)t_[i_++];
      if (c == '"') return out;
      if (c < 0x20) err("control character in string");
      if (c != '\\') {
        out += (char)c;
        continue;
      }
      if (i_ >= t_.size()) err("unterminated escape");
      const char e = t_[i_++];
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
            if (!(lit("\\u"))) err("unpaired surrogate");
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) err("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            err("unpaired surrogate");
          }
          utf8(out, cp);
          break;
        }
        default: err("bad escape");
      }
    }
  }
  JVal number() {
    const size_t s = i_;
    bool neg = false, frac = false;
    if (i_ < t_.size() && t_[i_] == '-') {
      neg = true;
      ++i_;
    }
    if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) err("invalid literal");
    if (t_[i_] == '0') {
      ++i_;
    } else {
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    if (i_ < t_.size() && t_[i_] == '.') {
      frac = true;
      ++i_;
      if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) err("invalid number");
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    if (i_ < t_.size() && (t_[i_] == 'e' || t_[i_] == 'E')) {
      frac = true;
      ++i_;
      if (i_ < t_.size() && (t_[i_] == '+' || t_[i_] == '-')) ++i_;
      if (i_ >= t_.size() || !(t_[i_] >= '0' && t_[i_] <= '9')) err("invalid number");
      while (i_ < t_.size() && t_[i_] >= '0' && t_[i_] <= '9') ++i_;
    }
    const std::string tok = t_.substr(s, i_ - s);
    JVal v;
    v.kind = JVal::NUM;
    v.num = std::strtod(tok.c_str(), nullptr);
    if (!neg && !frac) {
      errno = 0;
      const unsigned long long u = std::strtoull(tok.c_str(), nullptr, 10);
      if (errno == 0) {
        v.is_uint = true;
        v.u = u;
      }
    }
    return v;
  }
};

// Shortest round-trip digits of v laid out like the reference JSON library's
// dump (see the file header).
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string out;
  const char* p = buf;
  if (*p == '-') {
    out += '-';
    ++p;
  }
  std::string digits;
  while (*p && *p != 'e') {
    if (*p != '.') digits += *p;
    ++p;
  }
  const int e10 = std::atoi(p + 1);
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = (int)digits.size();
  const int n = e10 + 1;  // position of the decimal point
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int ex = n - 1;
    out += ex < 0 ? "e-" : "e+";
    const int a = ex < 0 ? -ex : ex;
    if (a < 10) out += '0';
    out += std::to_string(a);
  }
  return out;
}

const char* elem_name(int e) {
  switch (e) {
    case VK_ELEM_F32: return "f32";
    case VK_ELEM_U16: return "u16";
    case VK_ELEM_U32: return "u32";
    case VK_ELEM_BOOL: return "bool";
  }
  io_fail(VK_ERR_ARG, "unknown element kind");
}

uint64_t elem_bytes(int e) {
  switch (e) {
    case VK_ELEM_F32: return 4;
    case VK_ELEM_U16: return 2;
    case VK_ELEM_U32: return 4;
    case VK_ELEM_BOOL: return 1;
  }
  io_fail(VK_ERR_ARG, "unknown element kind");
}

const char* axes_for_rank(int rank) {  // io.cpp:33-41
  switch (rank) {
    case 1: return "X";
    case 2: return "YX";
    case 3: return "ZYX";
    case 4: return "CZYX";
  }
  bad_header("unsupported rank " + std::to_string(rank));
}

// Element count x element size; false when it does not fit in 64 bits (a
// crafted header could otherwise wrap to the real file size).
bool payload_bytes_checked(const vk_volume_info& info, uint64_t* out) {
  uint64_t n = 1;
  for (int a = 0; a < info.rank; ++a)
    if (__builtin_mul_overflow(n, info.shape[a], &n)) return false;
  return !__builtin_mul_overflow(n, (uint64_t)elem_bytes(info.elem), out);
}

uint64_t payload_bytes(const vk_volume_info& info) {
  uint64_t b = 0;
  if (!payload_bytes_checked(info, &b)) io_fail(VK_ERR_ARG, "volume too large (element count overflows)");
  return b;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

// io.cpp:83-131: magic, header length, JSON, required fields, elem, axes,
// payload length, trailing bytes; then the spacing (NdImage::with_spacing,
// image.cpp:197-205) as the reference attaches it after the payload checks.
vk_volume_info read_info(const char* path, File& file) {
  const std::string sp = path;
  file.f = std::fopen(path, "rb");
  if (!file.f) io_fail(VK_ERR_ARG, "cannot open '" + sp + "'");
  char magic[4];
  unsigned char len_le[4];
  if (std::fread(magic, 1, 4, file.f) != 4 || std::memcmp(magic, "NDIV", 4) != 0)
    io_fail(VK_ERR_BAD_MAGIC, "BadMagic: '" + sp + "' is not an NDIV volume");
  if (std::fread(len_le, 1, 4, file.f) != 4) bad_header("missing header length");
  const uint32_t len = (uint32_t)len_le[0] | ((uint32_t)len_le[1] << 8) | ((uint32_t)len_le[2] << 16) |
                       ((uint32_t)len_le[3] << 24);
  struct stat st {};
  if (fstat(fileno(file.f), &st) != 0) io_fail(VK_ERR_ARG, "cannot stat '" + sp + "'");
  // never allocate more header than the file holds
  if (8ull + len > (uint64_t)st.st_size) bad_header("truncated header");
  std::string head(len, '\0');
  if (len && std::fread(&head[0], 1, len, file.f) != len) bad_header("truncated header");
  const JVal h = JParser(head).document();
  if (h.kind != JVal::OBJ) bad_header("header is not valid JSON: expected an object");
  const JVal* je = h.find("elem");
  const JVal* js = h.find("shape");
  const JVal* ja = h.find("axes");
  if (!je || !js || !ja) bad_header("header needs elem, shape and axes");
  if (je->kind != JVal::STR) bad_header("elem must be a string");
  vk_volume_info info{};
  if (je->s == "f32") info.elem = VK_ELEM_F32;
  else if (je->s == "u16") info.elem = VK_ELEM_U16;
  else if (je->s == "u32") info.elem = VK_ELEM_U32;
  else if (je->s == "bool") info.elem = VK_ELEM_BOOL;
  else bad_header("unknown element kind '" + je->s + "'");
  if (js->kind != JVal::ARR) bad_header("shape must be an array of extents");
  if (js->arr.size() > VK_VOLUME_MAX_RANK) bad_header("unsupported rank " + std::to_string(js->arr.size()));
  for (const JVal& e : js->arr)
    if (e.kind != JVal::NUM || !e.is_uint) bad_header("shape must be an array of extents");
  if (ja->kind != JVal::STR) bad_header("axes must be a string");
  if (ja->s.size() != js->arr.size()) bad_header("axes string length must equal rank");
  info.rank = (int)js->arr.size();
  for (int a = 0; a < info.rank; ++a) info.shape[a] = js->arr[a].u;
  info.payload_offset = 8ull + len;
  if (!payload_bytes_checked(info, &info.payload_bytes)) bad_header("shape overflows the payload size");
  const uint64_t have = (uint64_t)st.st_size - std::min<uint64_t>((uint64_t)st.st_size, info.payload_offset);
  if (have < info.payload_bytes)
    truncated("expected " + std::to_string(info.payload_bytes) + " payload bytes in '" + sp + "'");
  if (have > info.payload_bytes) truncated("trailing bytes after payload in '" + sp + "'");
  if (const JVal* jsp = h.find("spacing")) {
    if (jsp->kind != JVal::ARR) bad_header("spacing must be an array");
    for (const JVal& e : jsp->arr)
      if (e.kind != JVal::NUM) bad_header("spacing must be an array of numbers");
    if ((int)jsp->arr.size() != info.rank)
      io_fail(VK_ERR_SHAPE, "ShapeMismatch: spacing needs one entry per axis");
    for (int a = 0; a < info.rank; ++a) {
      if (!(jsp->arr[a].num > 0.0)) io_fail(VK_ERR_SHAPE, "ShapeMismatch: spacing entries must be positive");
      info.spacing[a] = jsp->arr[a].num;
    }
    info.has_spacing = 1;
  }
  return info;
}

std::string header_json(const vk_volume_info& info) {
  // keys in sorted order, as the reference's std::map-backed object dumps them
  std::string h = "{\"axes\":\"";
  h += axes_for_rank(info.rank);
  h += "\",\"elem\":\"";
  h += elem_name(info.elem);
  h += "\",\"shape\":[";
  for (int a = 0; a < info.rank; ++a) {
    if (a) h += ',';
    h += std::to_string(info.shape[a]);
  }
  h += ']';
  if (info.has_spacing) {
    h += ",\"spacing\":[";
    for (int a = 0; a < info.rank; ++a) {
      if (a) h += ',';
      h += json_double(info.spacing[a]);
    }
    h += ']';
  }
  h += '}';
  return h;
}

void write_header(FILE* f, const std::string& path, const vk_volume_info& info) {
  const std::string h = header_json(info);
  const uint32_t len = (uint32_t)h.size();
  const unsigned char len_le[4] = {(unsigned char)(len & 0xff), (unsigned char)((len >> 8) & 0xff),
                                   (unsigned char)((len >> 16) & 0xff), (unsigned char)((len >> 24) & 0xff)};
  if (std::fwrite("NDIV", 1, 4, f) != 4 || std::fwrite(len_le, 1, 4, f) != 4 ||
      std::fwrite(h.data(), 1, h.size(), f) != h.size())
    io_fail(VK_ERR_ARG, "write to '" + path + "' failed");
}

void check_info_for_write(const vk_volume_info* info) {
  if (!info) io_fail(VK_ERR_ARG, "NULL argument");
  elem_name(info->elem);
  axes_for_rank(info->rank);  // HeaderMismatch before the file is touched (io.cpp:56)
}

// Two pinned staging buffers shared by every device transfer in the process.
constexpr size_t kChunk = 32u << 20;
struct Staging {
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int device = -1;
  void ensure() {
    int dev = 0;
    cuda_ck(cudaGetDevice(&dev), "cudaGetDevice");
    if (buf[0] && device == dev) return;
    for (int i = 0; i < 2; ++i) {
      if (!buf[i]) cuda_ck(cudaHostAlloc(&buf[i], kChunk, cudaHostAllocPortable), "pinned staging");
      if (ev[i]) cudaEventDestroy(ev[i]);
      cuda_ck(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
    }
    device = dev;
  }
};
Staging& staging() {
  static Staging* s = new Staging();  // process lifetime (pinned memory reused)
  return *s;
}

}  // namespace

extern "C" {

vk_status vk_volume_info_read(const char* path, vk_volume_info* info) {
  return io_guard([&] {
    if (!path || !info) io_fail(VK_ERR_ARG, "NULL argument");
    File f;
    *info = read_info(path, f);
  });
}

vk_status vk_volume_read(const char* path, vk_volume_info* info, void* dst, uint64_t dst_bytes) {
  return io_guard([&] {
    if (!path || !info) io_fail(VK_ERR_ARG, "NULL argument");
    File f;
    const vk_volume_info v = read_info(path, f);
    if (!dst || dst_bytes < v.payload_bytes) io_fail(VK_ERR_ARG, "destination buffer too small");
    if (v.payload_bytes && std::fread(dst, 1, v.payload_bytes, f.f) != v.payload_bytes)
      truncated("expected " + std::to_string(v.payload_bytes) + " payload bytes in '" + std::string(path) + "'");
    *info = v;
  });
}

vk_status vk_volume_read_device(const char* path, vk_volume_info* info, void* d_dst, uint64_t dst_bytes,
                                void* stream) {
  return io_guard([&] {
    if (!path || !info) io_fail(VK_ERR_ARG, "NULL argument");
    File f;
    const vk_volume_info v = read_info(path, f);
    if (!d_dst || dst_bytes < v.payload_bytes) io_fail(VK_ERR_ARG, "destination buffer too small");
    Staging& sg = staging();
    std::lock_guard<std::mutex> lock(sg.mu);
    sg.ensure();
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t off = 0;
    int k = 0;
    bool used[2] = {false, false};
    while (off < v.payload_bytes) {
      const size_t n = (size_t)std::min<uint64_t>(kChunk, v.payload_bytes - off);
      if (used[k]) cuda_ck(cudaEventSynchronize(sg.ev[k]), "staging wait");  // DMA out of buf[k] done
      if (std::fread(sg.buf[k], 1, n, f.f) != n)
        truncated("expected " + std::to_string(v.payload_bytes) + " payload bytes in '" + std::string(path) + "'");
      cuda_ck(cudaMemcpyAsync((char*)d_dst + off, sg.buf[k], n, cudaMemcpyHostToDevice, s), "H2D");
      cuda_ck(cudaEventRecord(sg.ev[k], s), "event");
      used[k] = true;
      off += n;
      k ^= 1;
    }
    for (int i = 0; i < 2; ++i)
      if (used[i]) cuda_ck(cudaEventSynchronize(sg.ev[i]), "staging wait");
    *info = v;
  });
}

vk_status vk_volume_write(const char* path, const vk_volume_info* info, const void* src) {
  return io_guard([&] {
    if (!path) io_fail(VK_ERR_ARG, "NULL argument");
    check_info_for_write(info);
    const std::string sp = path;
    const uint64_t bytes = payload_bytes(*info);
    if (bytes && !src) io_fail(VK_ERR_ARG, "NULL argument");
    File f;
    f.f = std::fopen(path, "wb");
    if (!f.f) io_fail(VK_ERR_ARG, "cannot open '" + sp + "' for writing");
    write_header(f.f, sp, *info);
    if (bytes && std::fwrite(src, 1, bytes, f.f) != bytes) io_fail(VK_ERR_ARG, "write to '" + sp + "' failed");
    const int rc = std::fclose(f.f);
    f.f = nullptr;
    if (rc != 0) io_fail(VK_ERR_ARG, "write to '" + sp + "' failed");
  });
}

vk_status vk_volume_write_device(const char* path, const vk_volume_info* info, const void* d_src, void* stream) {
  return io_guard([&] {
    if (!path) io_fail(VK_ERR_ARG, "NULL argument");
    check_info_for_write(info);
    const std::string sp = path;
    const uint64_t bytes = payload_bytes(*info);
    if (bytes && !d_src) io_fail(VK_ERR_ARG, "NULL argument");
    File f;
    f.f = std::fopen(path, "wb");
    if (!f.f) io_fail(VK_ERR_ARG, "cannot open '" + sp + "' for writing");
    write_header(f.f, sp, *info);
    Staging& sg = staging();
    std::lock_guard<std::mutex> lock(sg.mu);
    sg.ensure();
    cudaStream_t s = (cudaStream_t)stream;
    // chunk c goes through buf[c % 2]; D2H of chunk c+1 overlaps the write of c
    const uint64_t nchunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](uint64_t c) {
      const uint64_t off = c * kChunk;
      const size_t n = (size_t)std::min<uint64_t>(kChunk, bytes - off);
      cuda_ck(cudaMemcpyAsync(sg.buf[c & 1], (const char*)d_src + off, n, cudaMemcpyDeviceToHost, s), "D2H");
      cuda_ck(cudaEventRecord(sg.ev[c & 1], s), "event");
    };
    if (nchunks > 0) issue(0);
    if (nchunks > 1) issue(1);
    for (uint64_t c = 0; c < nchunks; ++c) {
      cuda_ck(cudaEventSynchronize(sg.ev[c & 1]), "staging wait");
      const size_t n = (size_t)std::min<uint64_t>(kChunk, bytes - c * kChunk);
      if (std::fwrite(sg.buf[c & 1], 1, n, f.f) != n) io_fail(VK_ERR_ARG, "write to '" + sp + "' failed");
      if (c + 2 < nchunks) issue(c + 2);
    }
    const int rc = std::fclose(f.f);
    f.f = nullptr;
    if (rc != 0) io_fail(VK_ERR_ARG, "write to '" + sp + "' failed");
  });
}

}  // extern "C"
