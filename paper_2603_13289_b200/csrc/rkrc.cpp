// rkrc.cpp -- the RKRC relay-cache file (relay_cache.cpp:176-253 over the
// serialize.cpp:45-117 container): "RKRC" | u32 version 1 | u64 manifest
// length | JSON manifest | fp32 blob, FNV-1a-64 checksum of the blob in the
// manifest. Files written here are byte-identical to the reference's
// export_relay_cache (the manifest reproduces nlohmann::json::dump(): sorted
// keys, compact separators, shortest round-trip floats), so caches move
// between the reference and the engine in both directions.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "rkrc.h"

namespace rk {
namespace {

uint64_t fnv1a64(const uint8_t* p, size_t n) {  // serialize.cpp:36-43
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

// nlohmann::json (3.11.3) number_float formatting, which the reference's
// manifest text goes through (serialize.cpp: json::dump): Grisu2 digit
// generation (F. Loitsch, "Printing Floating-Point Numbers Quickly and
// Accurately with Integers", PLDI 2010) with the boundaries of the double and
// the alpha/gamma window [-60, -32], then the format with min_exp -4 /
// max_exp 15: "10000.0", "0.0001", "1.5e-07", "803.1189575195313".
// Grisu2 does not always return the shortest/closest digits, so a shortest
// round-trip search would differ in the last digit for some floats
// (tests/test_rkrc.py sweeps 1,500 random thetas against the reference).
namespace grisu {
struct DiyFp {
  uint64_t f;
  int e;
};
DiyFp sub(DiyFp x, DiyFp y) { return {x.f - y.f, x.e}; }
DiyFp mul(DiyFp x, DiyFp y) {  // upper 64 bits of the 128-bit product, rounded half up
  const unsigned __int128 p = (unsigned __int128)x.f * y.f;
  const uint64_t h = (uint64_t)(p >> 64) + (uint64_t)((p >> 63) & 1);
  return {h, x.e + y.e + 64};
}
DiyFp normalize(DiyFp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    x.e--;
  }
  return x;
}
struct CachedPower {
  uint64_t f;
  int e, k;
};
// f * 2^e = 10^k rounded to nearest, f normalized to [2^63, 2^64), k = -300..324
// step 8 (generated exactly with Python Fractions).
constexpr CachedPower kPowers[] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324},
};
void round_last(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}
// digits of v (> 0, finite) into buf; value = buf * 10^dec_exp
void digits(double v, char* buf, int& len, int& dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  const uint64_t F = bits & ((1ull << 52) - 1), E = bits >> 52;
  const DiyFp w = E == 0 ? DiyFp{F, 1 - 1075} : DiyFp{F + (1ull << 52), (int)E - 1075};
  const bool closer = F == 0 && E > 1;  // the lower neighbour is half as far
  const DiyFp m_plus = normalize({2 * w.f + 1, w.e - 1});
  DiyFp m_minus = closer ? DiyFp{4 * w.f - 1, w.e - 2} : DiyFp{2 * w.f - 1, w.e - 1};
  m_minus = {m_minus.f << (m_minus.e - m_plus.e), m_plus.e};
  const DiyFp vn = normalize(w);
  // cached power c = 10^-k with alpha <= m_plus.e + c.e + 64 <= gamma
  const int f = -60 - m_plus.e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0);
  const CachedPower& cp = kPowers[(300 + k + 7) / 8];
  const DiyFp c{cp.f, cp.e};
  const DiyFp ww = mul(vn, c), wm = mul(m_minus, c), wp = mul(m_plus, c);
  const DiyFp Mm{wm.f + 1, wm.e}, Mp{wp.f - 1, wp.e};
  dec_exp = -cp.k;
  uint64_t delta = sub(Mp, Mm).f, dist = sub(Mp, ww).f;
  const DiyFp one{1ull << -Mp.e, Mp.e};
  uint32_t p1 = (uint32_t)(Mp.f >> -one.e);
  uint64_t p2 = Mp.f & (one.f - 1);
  uint32_t pow10 = 1;
  int n = 1;  // digits of p1
  for (uint32_t t = p1; t >= 10; t /= 10) {
    pow10 *= 10;
    ++n;
  }
  len = 0;
  while (n > 0) {
    const uint32_t d = p1 / pow10, r = p1 % pow10;
    buf[len++] = (char)('0' + d);
    p1 = r;
    --n;
    const uint64_t rest = ((uint64_t)p1 << -one.e) + p2;
    if (rest <= delta) {
      dec_exp += n;
      round_last(buf, len, dist, delta, rest, (uint64_t)pow10 << -one.e);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const uint64_t d = p2 >> -one.e, r = p2 & (one.f - 1);
    buf[len++] = (char)('0' + d);
    p2 = r;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  round_last(buf, len, dist, delta, p2, one.f);
}
}  // namespace grisu

std::string json_double(double v) {
  if (v == 0) return std::signbit(v) ? "-0.0" : "0.0";
  std::string out = v < 0 ? "-" : "";
  v = std::fabs(v);
  char buf[32];
  int len = 0, dec_exp = 0;
  grisu::digits(v, buf, len, dec_exp);
  const std::string digits(buf, buf + len);
  const int k = len, n = len + dec_exp;  // value = 0.digits * 10^n
  if (k <= n && n <= 15) {
    out += digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out += "0." + std::string(-n, '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int e = n - 1;
    char eb[8];
    std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', std::abs(e));
    out += eb;
  }
  return out;
}

// ---- minimal JSON reader for the manifest ----------------------------------
struct JVal {
  enum Kind { NUL, NUM, STR, ARR, OBJ, BOOL } kind = NUL;
  double num = 0;
  uint64_t u64 = 0;
  bool is_uint = false, neg = false;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct Parser {
  const char* p;
  const char* e;
  [[noreturn]] void fail(const std::string& m) { raise(RK_ERR_SCHEMA, "manifest parse error: " + m); }
  void ws() {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  JVal value() {
    ws();
    if (p >= e) fail("unexpected end");
    JVal v;
    if (*p == '{') {
      v.kind = JVal::OBJ;
      ++p;
      ws();
      if (p < e && *p == '}') { ++p; return v; }
      for (;;) {
        ws();
        JVal k = value();
        if (k.kind != JVal::STR) fail("object key");
        ws();
        if (p >= e || *p != ':') fail("':' expected");
        ++p;
        v.obj[k.str] = value();
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == '}') { ++p; break; }
        fail("',' or '}' expected");
      }
    } else if (*p == '[') {
      v.kind = JVal::ARR;
      ++p;
      ws();
      if (p < e && *p == ']') { ++p; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (p < e && *p == ',') { ++p; continue; }
        if (p < e && *p == ']') { ++p; break; }
        fail("',' or ']' expected");
      }
    } else if (*p == '"') {
      v.kind = JVal::STR;
      ++p;
      while (p < e && *p != '"') {
        if (*p == '\\') {
          ++p;
          if (p >= e) fail("escape");
        }
        v.str += *p++;
      }
      if (p >= e) fail("unterminated string");
      ++p;
    } else if (std::strncmp(p, "null", 4) == 0) {
      p += 4;
    } else if (std::strncmp(p, "true", 4) == 0 || std::strncmp(p, "false", 5) == 0) {
      v.kind = JVal::BOOL;
      v.num = *p == 't';
      p += *p == 't' ? 4 : 5;
    } else {
      v.kind = JVal::NUM;
      const char* s = p;
      if (*p == '-') { v.neg = true; ++p; }
      bool integral = true;
      while (p < e && (std::isdigit((unsigned char)*p) || *p == '.' || *p == 'e' || *p == 'E' || *p == '+' ||
                       *p == '-')) {
        if (*p == '.' || *p == 'e' || *p == 'E') integral = false;
        ++p;
      }
      const std::string t(s, p);
      if (t.empty() || t == "-") fail("number");
      v.num = std::strtod(t.c_str(), nullptr);
      if (integral && !v.neg) {
        v.is_uint = true;
        v.u64 = std::strtoull(t.c_str(), nullptr, 10);
      }
    }
    return v;
  }
};

const JVal& at(const JVal& o, const char* k) {
  auto it = o.obj.find(k);
  if (o.kind != JVal::OBJ || it == o.obj.end()) raise(RK_ERR_SCHEMA, std::string("relay cache manifest: key '") + k + "' not found");
  return it->second;
}
uint64_t as_u64(const JVal& v, const char* what) {
  if (v.kind != JVal::NUM || !v.is_uint) raise(RK_ERR_SCHEMA, std::string("relay cache manifest: ") + what + " must be an unsigned integer");
  return v.u64;
}

}  // namespace

std::vector<uint8_t> rkrc_encode(const rk_relay_cache_view& c) {
  const uint64_t L = c.num_layers, n = c.segment_len, kv = c.num_kv_heads * c.d_head, d = c.d_model;
  // blob in export order: k_pre.l, v.l per layer, hidden_snapshot, influence
  std::vector<uint8_t> blob;
  blob.reserve((2 * L * n * kv + n * d + n) * 4);
  std::string tensors = "[";
  auto add = [&](const std::string& name, const float* data, std::vector<uint64_t> shape) {
    uint64_t count = 1;
    for (uint64_t s : shape) count *= s;
    if (tensors.size() > 1) tensors += ",";
    tensors += "{\"name\":\"" + name + "\",\"offset\":" + std::to_string(blob.size()) + ",\"shape\":[";
    for (size_t i = 0; i < shape.size(); ++i) tensors += (i ? "," : "") + std::to_string(shape[i]);
    tensors += "]}";
    const uint8_t* b = reinterpret_cast<const uint8_t*>(data);
    blob.insert(blob.end(), b, b + count * 4);
  };
  for (uint64_t l = 0; l < L; ++l) {
    add("k_pre." + std::to_string(l), c.k_pre[l], {n, kv});
    add("v." + std::to_string(l), c.v[l], {n, kv});
  }
  add("hidden_snapshot", c.hidden_snapshot, {n, d});
  add("influence", c.influence, {n});
  tensors += "]";
  std::string toks = "[";
  for (uint64_t i = 0; i < n; ++i) toks += (i ? "," : "") + std::to_string(c.segment_tokens[i]);
  toks += "]";
  // nlohmann::json object keys are sorted (std::map)
  const std::string m = "{\"blob_bytes\":" + std::to_string(blob.size()) +
                        ",\"blob_checksum\":" + std::to_string(fnv1a64(blob.data(), blob.size())) +
                        ",\"d_head\":" + std::to_string(c.d_head) + ",\"d_model\":" + std::to_string(d) +
                        ",\"decode_steps_observed\":" + std::to_string(c.decode_steps_observed) +
                        ",\"kind\":\"relay-cache\",\"max_positions\":" + std::to_string(c.max_positions) +
                        ",\"num_kv_heads\":" + std::to_string(c.num_kv_heads) + ",\"num_layers\":" + std::to_string(L) +
                        ",\"schema_version\":1,\"segment_tokens\":" + toks +
                        ",\"snapshot_layer\":" + std::to_string(c.snapshot_layer) +
                        ",\"source_base_position\":" + std::to_string(c.source_base_position) + ",\"tensors\":" + tensors +
                        ",\"theta_base\":" + json_double((double)c.theta_base) + "}";
  std::vector<uint8_t> out;
  out.reserve(16 + m.size() + blob.size());
  out.insert(out.end(), {'R', 'K', 'R', 'C'});
  const uint32_t version = 1;  // kBlobFormatVersion (serialize.hpp:25)
  const uint64_t mlen = m.size();
  out.insert(out.end(), reinterpret_cast<const uint8_t*>(&version), reinterpret_cast<const uint8_t*>(&version) + 4);
  out.insert(out.end(), reinterpret_cast<const uint8_t*>(&mlen), reinterpret_cast<const uint8_t*>(&mlen) + 8);
  out.insert(out.end(), m.begin(), m.end());
  out.insert(out.end(), blob.begin(), blob.end());
  return out;
}

void rkrc_write(const std::string& path, const std::vector<uint8_t>& bytes) {
  std::ofstream f(path, std::ios::binary);
  if (!f) raise(RK_ERR_IO, "cannot open for writing: " + path);
  f.write(reinterpret_cast<const char*>(bytes.data()), (std::streamsize)bytes.size());
  if (!f) raise(RK_ERR_IO, "write failed: " + path);
}

namespace {
// A byte source: a file (blob read straight into the destination buffer) or memory.
struct Source {
  uint64_t size = 0;
  std::FILE* f = nullptr;
  const uint8_t* mem = nullptr;
  uint64_t pos = 0;
  std::string name;
  void read(void* dst, uint64_t n) {
    if (f) {
      if (std::fread(dst, 1, n, f) != n) raise(RK_ERR_IO, "read failed: " + name);
    } else {
      std::memcpy(dst, mem + pos, n);
    }
    pos += n;
  }
};
HostCacheFile decode(Source& src, bool pinned);
}  // namespace

HostCacheFile rkrc_read(const std::string& path, bool pinned) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) raise(RK_ERR_IO, "cannot open: " + path);
  struct Closer {
    std::FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{f};
  std::fseek(f, 0, SEEK_END);
  Source src;
  src.size = (uint64_t)std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  src.f = f;
  src.name = path;
  return decode(src, pinned);
}

HostCacheFile rkrc_decode(const uint8_t* bytes, uint64_t size) {
  Source src;
  src.mem = bytes;
  src.size = size;
  return decode(src, false);
}

namespace {
HostCacheFile decode(Source& src, bool pinned) {
  const uint64_t size = src.size;
  // BlobReader::from_bytes (serialize.cpp:84-117)
  uint8_t hdr[16];
  if (size < 16) raise(RK_ERR_SCHEMA, "blob file truncated (header)");
  src.read(hdr, 16);
  if (std::memcmp(hdr, "RKRC", 4) != 0) raise(RK_ERR_SCHEMA, "bad magic, expected 'RKRC'");
  uint32_t version;
  uint64_t mlen;
  std::memcpy(&version, hdr + 4, 4);
  std::memcpy(&mlen, hdr + 8, 8);
  if (version != 1) raise(RK_ERR_SCHEMA, "unsupported format version " + std::to_string(version));
  if (mlen > size - 16) raise(RK_ERR_SCHEMA, "blob file truncated (manifest)");  // (no 16 + mlen wrap)
  std::string mtext(mlen, '\0');
  src.read(mtext.data(), mlen);
  Parser ps{mtext.data(), mtext.data() + mlen};
  const JVal m = ps.value();
  HostCacheFile h;
  // the blob goes straight into its own (optionally pinned) aligned buffer
  h.blob_size = size - 16 - mlen;
  h.alloc(h.blob_size, pinned);
  if (h.blob_size) src.read(h.blob.get(), h.blob_size);
  const uint8_t* blob = h.blob.get();
  if (m.kind != JVal::OBJ || !m.obj.count("blob_bytes") || !m.obj.count("blob_checksum"))
    raise(RK_ERR_SCHEMA, "manifest missing blob_bytes/blob_checksum");
  if (as_u64(at(m, "blob_bytes"), "blob_bytes") != h.blob_size)
    raise(RK_ERR_SCHEMA, "blob truncated: manifest declares " + std::to_string(at(m, "blob_bytes").u64) +
                             " bytes, file has " + std::to_string(h.blob_size));
  if (as_u64(at(m, "blob_checksum"), "blob_checksum") != fnv1a64(blob, h.blob_size))
    raise(RK_ERR_SCHEMA, "blob checksum mismatch");
  // import_relay_cache (relay_cache.cpp:203-236)
  rk_relay_cache_view& c = h.view;
  c.num_kv_heads = as_u64(at(m, "num_kv_heads"), "num_kv_heads");
  c.d_head = as_u64(at(m, "d_head"), "d_head");
  c.d_model = as_u64(at(m, "d_model"), "d_model");
  const JVal& theta = at(m, "theta_base");
  if (theta.kind != JVal::NUM) raise(RK_ERR_SCHEMA, "relay cache manifest: theta_base must be a number");
  c.theta_base = (float)theta.num;
  c.max_positions = as_u64(at(m, "max_positions"), "max_positions");
  c.source_base_position = as_u64(at(m, "source_base_position"), "source_base_position");
  c.snapshot_layer = as_u64(at(m, "snapshot_layer"), "snapshot_layer");
  c.decode_steps_observed = as_u64(at(m, "decode_steps_observed"), "decode_steps_observed");
  const JVal& toks = at(m, "segment_tokens");
  if (toks.kind != JVal::ARR) raise(RK_ERR_SCHEMA, "relay cache manifest: segment_tokens must be an array");
  for (const JVal& t : toks.arr) {
    if (t.kind != JVal::NUM || t.num != std::floor(t.num))
      raise(RK_ERR_SCHEMA, "relay cache manifest: token ids must be integers");
    h.tokens.push_back((int32_t)t.num);
  }
  const uint64_t L = as_u64(at(m, "num_layers"), "num_layers");
  c.num_layers = L;
  c.segment_len = h.tokens.size();
  const JVal& recs = at(m, "tensors");
  auto get = [&](const std::string& name, std::vector<uint64_t>* shape) -> const float* {  // BlobReader::get
    for (const JVal& r : recs.arr) {
      if (at(r, "name").str != name) continue;
      uint64_t count = 1;
      shape->clear();
      for (const JVal& s : at(r, "shape").arr) {
        shape->push_back(as_u64(s, "shape"));
        count *= shape->back();
      }
      const uint64_t off = as_u64(at(r, "offset"), "offset");
      if (off + count * 4 > h.blob_size) raise(RK_ERR_SCHEMA, "tensor '" + name + "' extends past end of blob");
      if (off % 4) raise(RK_ERR_SCHEMA, "tensor '" + name + "' is not 4-byte aligned in the blob");
      return reinterpret_cast<const float*>(blob + off);
    }
    raise(RK_ERR_SCHEMA, "tensor '" + name + "' not found in manifest");
  };
  // RelayCache::validate (relay_cache.cpp:18-41), errors prefixed like import
  auto bad = [](const std::string& what) { raise(RK_ERR_SCHEMA, "relay cache file: relay cache: " + what); };
  const uint64_t n = c.segment_len, kv = c.num_kv_heads * c.d_head;
  std::vector<uint64_t> shk, shv;
  h.k.resize(L);
  h.v.resize(L);
  for (uint64_t l = 0; l < L; ++l) {
    h.k[l] = get("k_pre." + std::to_string(l), &shk);
    h.v[l] = get("v." + std::to_string(l), &shv);
    const std::vector<uint64_t> want{n, kv};
    if (shk != want || shv != want) bad("layer " + std::to_string(l) + " tensor shape mismatch");
  }
  if (n == 0) bad("empty segment");
  if (L == 0) bad("per-layer K/V tables disagree");
  if (c.snapshot_layer >= L) bad("snapshot layer out of range");
  std::vector<uint64_t> shh, shi;
  c.hidden_snapshot = get("hidden_snapshot", &shh);
  if (shh != std::vector<uint64_t>{n, c.d_model}) bad("hidden snapshot shape mismatch");
  c.influence = get("influence", &shi);
  uint64_t ni = 1;
  for (uint64_t s : shi) ni *= s;
  if (ni != n) bad("influence length mismatch");
  for (uint64_t j = 0; j < n; ++j)
    if (!(c.influence[j] >= 0.0f)) bad("negative influence score");
  c.k_pre = h.k.data();
  c.v = h.v.data();
  c.segment_tokens = h.tokens.data();
  return h;
}
}  // namespace

void HostCacheFile::alloc(uint64_t bytes, bool pinned) {
  void* p = nullptr;
  if (pinned) {
    if (cudaMallocHost(&p, bytes ? bytes : 4) != cudaSuccess) {
      cudaGetLastError();
      raise(RK_ERR_RUNTIME, "cudaMallocHost failed for " + std::to_string(bytes) + " bytes");
    }
    blob = std::shared_ptr<uint8_t>(static_cast<uint8_t*>(p), [](uint8_t* q) { cudaFreeHost(q); });
  } else {
    p = std::malloc(bytes ? bytes : 4);
    if (!p) raise(RK_ERR_RUNTIME, "out of host memory");
    blob = std::shared_ptr<uint8_t>(static_cast<uint8_t*>(p), [](uint8_t* q) { std::free(q); });
  }
}

}  // namespace rk
