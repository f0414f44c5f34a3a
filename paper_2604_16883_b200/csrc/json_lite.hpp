// json_lite.hpp — the small JSON reader/writer the host side needs for the
// reference's two JSON artefacts: threshold profiles (calibration.cpp:174-243,
// schema SPEC.md "Profile JSON schema") and snapshot manifests
// (kv_cache.cpp:123-191).  The reference uses nlohmann/json (unpinned); files
// written by either side parse on the other: numbers are written with 17
// significant digits (exact double round trip) and read with strtod.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace sinkr {
namespace json {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;                    // String, or the literal text of a Number
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;  // insertion order

    bool is_number() const { return kind == Number; }
    bool is_array() const { return kind == Array; }
    bool is_object() const { return kind == Object; }
    bool contains(const std::string& k) const {
        if (kind != Object) return false;
        for (const auto& kv : obj)
            if (kv.first == k) return true;
        return false;
    }
    const Value& at(const std::string& k) const {
        if (kind == Object)
            for (const auto& kv : obj)
                if (kv.first == k) return kv.second;
        throw std::runtime_error("JSON key \"" + k + "\" not found");
    }
    double as_double() const {
        if (kind != Number) throw std::runtime_error("JSON value is not a number");
        return num;
    }
    unsigned long long as_u64() const {
        if (kind != Number) throw std::runtime_error("JSON value is not a number");
        if (str.find_first_of(".eE-") != std::string::npos) {
            if (num < 0 || num != (double)(unsigned long long)num)
                throw std::runtime_error("JSON value is not an unsigned integer");
            return (unsigned long long)num;
        }
        return std::strtoull(str.c_str(), nullptr, 10);
    }
    long long as_i64() const {
        if (kind != Number) throw std::runtime_error("JSON value is not a number");
        if (str.find_first_of(".eE") != std::string::npos) return (long long)num;
        return std::strtoll(str.c_str(), nullptr, 10);
    }
};

class Parser {
  public:
    explicit Parser(const std::string& text) : s_(text) {}
    Value parse() {
        Value v = value();
        ws();
        if (i_ != s_.size()) error("trailing characters");
        return v;
    }

  private:
    const std::string& s_;
    size_t i_ = 0;

    [[noreturn]] void error(const std::string& what) const {
        throw std::runtime_error("JSON parse error at offset " + std::to_string(i_) + ": " + what);
    }
    void ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
            ++i_;
    }
    bool lit(const char* w) {
        size_t n = 0;
        while (w[n]) ++n;
        if (s_.compare(i_, n, w) == 0) {
            i_ += n;
            return true;
        }
        return false;
    }
    Value value() {
        ws();
        if (i_ >= s_.size()) error("unexpected end of input");
        const char c = s_[i_];
        Value v;
        if (c == '{') {
            v.kind = Value::Object;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == '}') {
                ++i_;
                return v;
            }
            for (;;) {
                ws();
                if (i_ >= s_.size() || s_[i_] != '"') error("expected object key");
                std::string k = string();
                ws();
                if (i_ >= s_.size() || s_[i_] != ':') error("expected ':'");
                ++i_;
                v.obj.emplace_back(std::move(k), value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == '}') {
                    ++i_;
                    return v;
                }
                error("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = Value::Array;
            ++i_;
            ws();
            if (i_ < s_.size() && s_[i_] == ']') {
                ++i_;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (i_ < s_.size() && s_[i_] == ',') {
                    ++i_;
                    continue;
                }
                if (i_ < s_.size() && s_[i_] == ']') {
                    ++i_;
                    return v;
                }
                error("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = Value::String;
            v.str = string();
            return v;
        }
        if (lit("true")) {
            v.kind = Value::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = Value::Bool;
            return v;
        }
        if (lit("null")) return v;
        if (c == '-' || (c >= '0' && c <= '9')) {
            const size_t b = i_;
            if (s_[i_] == '-') ++i_;
            while (i_ < s_.size() && ((s_[i_] >= '0' && s_[i_] <= '9') || s_[i_] == '.' ||
                                      s_[i_] == 'e' || s_[i_] == 'E' || s_[i_] == '+' || s_[i_] == '-'))
                ++i_;
            v.kind = Value::Number;
            v.str = s_.substr(b, i_ - b);
            char* end = nullptr;
            v.num = std::strtod(v.str.c_str(), &end);
            if (!end || *end) error("bad number '" + v.str + "'");
            return v;
        }
        error(std::string("unexpected character '") + c + "'");
    }
    std::string string() {
        std::string out;
        ++i_;  // opening quote
        while (i_ < s_.size() && s_[i_] != '"') {
            char c = s_[i_++];
            if (c == '\\') {
                if (i_ >= s_.size()) error("bad escape");
                const char e = s_[i_++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (i_ + 4 > s_.size()) error("bad \\u escape");
                        const unsigned cp = (unsigned)std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16);
                        i_ += 4;
                        if (cp < 0x80) {
                            out += (char)cp;
                        } else if (cp < 0x800) {
                            out += (char)(0xC0 | (cp >> 6));
                            out += (char)(0x80 | (cp & 0x3F));
                        } else {
                            out += (char)(0xE0 | (cp >> 12));
                            out += (char)(0x80 | ((cp >> 6) & 0x3F));
                            out += (char)(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: out += e;
                }
            } else {
                out += c;
            }
        }
        if (i_ >= s_.size()) error("unterminated string");
        ++i_;
        return out;
    }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

// 17 significant digits: every double survives a write/read round trip.
inline std::string num(double x) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.17g", x);
    std::string s(buf);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // keep it a float literal
    return s;
}
inline std::string num(unsigned long long x) { return std::to_string(x); }

inline std::string quote(const std::string& s) {
    std::string out = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') {
            out += '\\';
            out += c;
        } else if (c == '\n') {
            out += "\\n";
        } else {
            out += c;
        }
    }
    return out + "\"";
}

}  // namespace json
}  // namespace sinkr
