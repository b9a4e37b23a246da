// ref_shim.cpp -- C entry points onto the REFERENCE's own core library, compiled from
// the sources where they lie under /root/reference/proj (oracle/Makefile target `ref`,
// output in oracle/_ref/).  Test infrastructure only: used by tests/test_frame_ref.py
// to pin the ISF1 frame bytes (proj/src/core/frame.cpp:9-71) and the Field/Error
// conventions (proj/src/core/types.cpp:37-74, proj/include/isf/core/errors.hpp:43-52).
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "isf/core/crc32.hpp"
#include "isf/core/errors.hpp"
#include "isf/core/frame.hpp"
#include "isf/core/types.hpp"

namespace {
thread_local std::string g_msg;
int code_of(const isf::Error& e) { return 1 + static_cast<int>(e.code()); }
}  // namespace

extern "C" {

const char* ref_last_message() { return g_msg.c_str(); }

// build_frame(header, payload) -> bytes written to out (cap bytes); returns frame length or 0
unsigned long long ref_build_frame(unsigned kind, unsigned long long step, double sim_time, unsigned E, unsigned P,
                                   unsigned comps, const unsigned char* payload, unsigned long long n,
                                   unsigned char* out, unsigned long long cap) {
  isf::FrameHeader h;
  h.kind = static_cast<isf::PayloadKind>(kind);
  h.step_index = step;
  h.sim_time = sim_time;
  h.elements_per_axis = E;
  h.points_per_element_axis = P;
  h.components = comps;
  auto b = isf::build_frame(h, {reinterpret_cast<const std::byte*>(payload), (size_t)n});
  if (b.size() > cap) return 0;
  std::memcpy(out, b.data(), b.size());
  return b.size();
}

// parse_frame: returns 0 and the payload offset/length, or 1 + ErrorCode
int ref_parse_frame(const unsigned char* frame, unsigned long long n, unsigned long long* payload_off,
                    unsigned long long* payload_len, unsigned* kind) {
  try {
    auto pf = isf::parse_frame({reinterpret_cast<const std::byte*>(frame), (size_t)n});
    *payload_off = (unsigned long long)(reinterpret_cast<const unsigned char*>(pf.payload.data()) - frame);
    *payload_len = pf.payload.size();
    *kind = static_cast<unsigned>(pf.header.kind);
    return 0;
  } catch (const isf::Error& e) {
    g_msg = e.what();
    return code_of(e);
  }
}

unsigned ref_crc32(const unsigned char* p, unsigned long long n) {
  return isf::crc32_ieee({reinterpret_cast<const std::byte*>(p), (size_t)n});
}

// Field::validate via the constructor: 0 or 1 + ErrorCode
int ref_field_validate(unsigned E, unsigned P, unsigned comps, const double* v, unsigned long long n) {
  try {
    isf::Field f(E, P, comps, std::vector<double>(v, v + n));
    (void)f;
    return 0;
  } catch (const isf::Error& e) {
    g_msg = e.what();
    return code_of(e);
  }
}

const char* ref_error_code_name(int code) { return isf::error_code_name(static_cast<isf::ErrorCode>(code)); }
}
