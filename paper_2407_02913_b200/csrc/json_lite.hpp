// Minimal JSON value for the drop-in's file formats (SFCT headers, layer lists,
// run manifests, CLI reports).  The reference serialises these with a vendored
// JSON library that is absent here; what matters for a drop-in is the text it
// writes, so dump() reproduces that library's conventions:
//   * objects keep their keys sorted (std::map),
//   * dump() is compact, dump(n) puts every member / element on its own line,
//     indented n spaces per level, with ": " after keys,
//   * doubles print as the shortest round-trip digits laid out with a decimal
//     point between 1e-5 and 1e15 ("1000.0", "0.001"), exponent form outside it
//     ("1e-05", "1.5e+16"); NaN and infinities print as null,
//   * integers print in full, strings escape '"', '\\' and control characters.
// parse() accepts RFC 8259 text; numbers without '.', 'e' or 'E' become integers
// (unsigned when non-negative), like that library.  Errors throw std::runtime_error.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace sfcb200 {
namespace json {

class Value {
public:
    enum class Kind { Null, Bool, Int, UInt, Float, String, Array, Object };

    Value() = default;
    Value(std::nullptr_t) {}
    Value(bool b) : kind_(Kind::Bool), b_(b) {}
    Value(int v) : kind_(Kind::Int), i_(v) {}
    Value(long v) : kind_(Kind::Int), i_(v) {}
    Value(long long v) : kind_(Kind::Int), i_(v) {}
    Value(unsigned v) : kind_(Kind::UInt), u_(v) {}
    Value(unsigned long v) : kind_(Kind::UInt), u_(v) {}
    Value(unsigned long long v) : kind_(Kind::UInt), u_(v) {}
    Value(double v) : kind_(Kind::Float), f_(v) {}
    Value(const char* s) : kind_(Kind::String), s_(s) {}
    Value(std::string s) : kind_(Kind::String), s_(std::move(s)) {}

    static Value array() { Value v; v.kind_ = Kind::Array; return v; }
    static Value object() { Value v; v.kind_ = Kind::Object; return v; }

    Kind kind() const { return kind_; }
    bool is_array() const { return kind_ == Kind::Array; }
    bool is_object() const { return kind_ == Kind::Object; }
    bool is_number() const { return kind_ == Kind::Int || kind_ == Kind::UInt || kind_ == Kind::Float; }
    bool is_string() const { return kind_ == Kind::String; }

    // object access; operator[] turns a null value into an object
    Value& operator[](const std::string& key) {
        if (kind_ == Kind::Null) kind_ = Kind::Object;
        if (kind_ != Kind::Object) throw std::runtime_error("json: cannot index a non-object with '" + key + "'");
        return obj_[key];
    }
    const Value& at(const std::string& key) const {
        if (kind_ != Kind::Object) throw std::runtime_error("json: cannot look up '" + key + "' in a non-object");
        auto it = obj_.find(key);
        if (it == obj_.end()) throw std::runtime_error("json: key '" + key + "' not found");
        return it->second;
    }
    bool contains(const std::string& key) const { return kind_ == Kind::Object && obj_.count(key) != 0; }
    void push_back(Value v) {
        if (kind_ == Kind::Null) kind_ = Kind::Array;
        if (kind_ != Kind::Array) throw std::runtime_error("json: push_back on a non-array");
        arr_.push_back(std::move(v));
    }
    const std::vector<Value>& items() const {
        if (kind_ != Kind::Array) throw std::runtime_error("json: not an array");
        return arr_;
    }
    bool empty() const { return kind_ == Kind::Array ? arr_.empty() : kind_ == Kind::Object ? obj_.empty() : false; }

    // conversions (numbers convert between kinds like a static_cast)
    long long as_int() const {
        switch (kind_) {
            case Kind::Int: return i_;
            case Kind::UInt: return static_cast<long long>(u_);
            case Kind::Float: return static_cast<long long>(f_);
            default: throw std::runtime_error("json: type must be number, but is " + kind_name());
        }
    }
    unsigned long long as_uint() const {
        switch (kind_) {
            case Kind::Int: return static_cast<unsigned long long>(i_);
            case Kind::UInt: return u_;
            case Kind::Float: return static_cast<unsigned long long>(f_);
            default: throw std::runtime_error("json: type must be number, but is " + kind_name());
        }
    }
    double as_double() const {
        switch (kind_) {
            case Kind::Int: return double(i_);
            case Kind::UInt: return double(u_);
            case Kind::Float: return f_;
            default: throw std::runtime_error("json: type must be number, but is " + kind_name());
        }
    }
    const std::string& as_string() const {
        if (kind_ != Kind::String) throw std::runtime_error("json: type must be string, but is " + kind_name());
        return s_;
    }
    std::string kind_name() const {
        static const char* names[] = {"null", "boolean", "number", "number", "number", "string", "array", "object"};
        return names[int(kind_)];
    }

    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

    static Value parse(const std::string& text);

private:
    static void write_string(std::string& out, const std::string& s) {
        out += '"';
        for (unsigned char c : s) {
            switch (c) {
                case '"': out += "\\\""; break;
                case '\\': out += "\\\\"; break;
                case '\b': out += "\\b"; break;
                case '\f': out += "\\f"; break;
                case '\n': out += "\\n"; break;
                case '\r': out += "\\r"; break;
                case '\t': out += "\\t"; break;
                default:
                    if (c < 0x20) {
                        char buf[8];
                        std::snprintf(buf, sizeof buf, "\\u%04x", unsigned(c));
                        out += buf;
                    } else {
                        out += char(c);
                    }
            }
        }
        out += '"';
    }

    static void write_double(std::string& out, double v) {
        if (!std::isfinite(v)) {
            out += "null";
            return;
        }
        if (v == 0.0) {
            out += std::signbit(v) ? "-0.0" : "0.0";
            return;
        }
        // shortest round-trip digits d.ddd e X  ->  digits D (k of them), point position n = X + 1
        char buf[64];
        auto res = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
        std::string sci(buf, res.ptr);
        std::string sign;
        if (sci[0] == '-') sign = "-", sci.erase(0, 1);
        const size_t epos = sci.find('e');
        std::string digits = sci.substr(0, epos);
        if (digits.size() > 1) digits.erase(1, 1);  // drop the '.'
        const int n = std::stoi(sci.substr(epos + 1)) + 1;
        const int k = int(digits.size());
        out += sign;
        if (k <= n && n <= 15) {
            out += digits + std::string(size_t(n - k), '0') + ".0";
        } else if (0 < n && n <= 15) {
            out += digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
        } else if (-4 < n && n <= 0) {
            out += "0." + std::string(size_t(-n), '0') + digits;
        } else {
            out += digits.substr(0, 1);
            if (k > 1) out += "." + digits.substr(1);
            const int e = n - 1;
            char eb[16];
            std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
            out += eb;
        }
    }

    void write(std::string& out, int indent, int level) const {
        const bool pretty = indent >= 0;
        auto pad = [&](int lv) {
            if (pretty) out.append(size_t(lv) * size_t(indent), ' ');
        };
        switch (kind_) {
            case Kind::Null: out += "null"; break;
            case Kind::Bool: out += b_ ? "true" : "false"; break;
            case Kind::Int: out += std::to_string(i_); break;
            case Kind::UInt: out += std::to_string(u_); break;
            case Kind::Float: write_double(out, f_); break;
            case Kind::String: write_string(out, s_); break;
            case Kind::Array:
                if (arr_.empty()) {
                    out += "[]";
                    break;
                }
                out += pretty ? "[\n" : "[";
                for (size_t i = 0; i < arr_.size(); ++i) {
                    pad(level + 1);
                    arr_[i].write(out, indent, level + 1);
                    if (i + 1 < arr_.size()) out += pretty ? ",\n" : ",";
                }
                if (pretty) out += "\n";
                pad(level);
                out += "]";
                break;
            case Kind::Object: {
                if (obj_.empty()) {
                    out += "{}";
                    break;
                }
                out += pretty ? "{\n" : "{";
                size_t i = 0;
                for (const auto& kv : obj_) {
                    pad(level + 1);
                    write_string(out, kv.first);
                    out += pretty ? ": " : ":";
                    kv.second.write(out, indent, level + 1);
                    if (++i < obj_.size()) out += pretty ? ",\n" : ",";
                }
                if (pretty) out += "\n";
                pad(level);
                out += "}";
                break;
            }
        }
    }

    Kind kind_ = Kind::Null;
    bool b_ = false;
    long long i_ = 0;
    unsigned long long u_ = 0;
    double f_ = 0.0;
    std::string s_;
    std::vector<Value> arr_;
    std::map<std::string, Value> obj_;

    friend class Parser;
};

class Parser {
public:
    explicit Parser(const std::string& t) : t_(t) {}

    Value document() {
        Value v = value(0);
        ws();
        if (p_ != t_.size()) fail("unexpected trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const std::string& what) const {
        throw std::runtime_error("json parse error at byte " + std::to_string(p_) + ": " + what);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < t_.size() && t_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    bool literal(const char* word) {
        const std::string w(word);
        if (t_.compare(p_, w.size(), w) == 0) {
            p_ += w.size();
            return true;
        }
        return false;
    }

    Value value(int depth) {
        if (depth > 512) fail("nesting too deep");
        ws();
        if (p_ >= t_.size()) fail("unexpected end of input");
        const char c = t_[p_];
        if (c == '{') {
            ++p_;
            Value o = Value::object();
            if (eat('}')) return o;
            do {
                ws();
                if (p_ >= t_.size() || t_[p_] != '"') fail("expected a string key");
                std::string k = string();
                expect(':');
                o.obj_[k] = value(depth + 1);
            } while (eat(','));
            expect('}');
            return o;
        }
        if (c == '[') {
            ++p_;
            Value a = Value::array();
            if (eat(']')) return a;
            do a.arr_.push_back(value(depth + 1));
            while (eat(','));
            expect(']');
            return a;
        }
        if (c == '"') return Value(string());
        if (literal("true")) return Value(true);
        if (literal("false")) return Value(false);
        if (literal("null")) return Value();
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        fail(std::string("unexpected character '") + c + "'");
    }

    static void utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) {
            out += char(cp);
        } else if (cp < 0x800) {
            out += char(0xC0 | (cp >> 6)), out += char(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += char(0xE0 | (cp >> 12)), out += char(0x80 | ((cp >> 6) & 0x3F)), out += char(0x80 | (cp & 0x3F));
        } else {
            out += char(0xF0 | (cp >> 18)), out += char(0x80 | ((cp >> 12) & 0x3F));
            out += char(0x80 | ((cp >> 6) & 0x3F)), out += char(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (p_ + 4 > t_.size()) fail("truncated \\u escape");
        unsigned v = 0;
        for (int i = 0; i < 4; ++i) {
            const char h = t_[p_++];
            v <<= 4;
            if (h >= '0' && h <= '9') v |= unsigned(h - '0');
            else if (h >= 'a' && h <= 'f') v |= unsigned(h - 'a' + 10);
            else if (h >= 'A' && h <= 'F') v |= unsigned(h - 'A' + 10);
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        while (true) {
            if (p_ >= t_.size()) fail("unterminated string");
            const unsigned char c = static_cast<unsigned char>(t_[p_++]);
            if (c == '"') return out;
            if (c < 0x20) fail("control character in string");
            if (c != '\\') {
                out += char(c);
                continue;
            }
            if (p_ >= t_.size()) fail("unterminated escape");
            const char e = t_[p_++];
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
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00) {
                        if (t_.compare(p_, 2, "\\u") != 0) fail("lone surrogate");
                        p_ += 2;
                        const unsigned lo = hex4();
                        if (lo < 0xDC00 || lo > 0xDFFF) fail("bad surrogate pair");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    utf8(out, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
    }
    Value number() {
        const size_t start = p_;
        bool is_float = false;
        if (t_[p_] == '-') ++p_;
        auto digits = [&] {
            const size_t s = p_;
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
            if (p_ == s) fail("expected digits");
        };
        if (p_ < t_.size() && t_[p_] == '0') ++p_;
        else digits();
        if (p_ < t_.size() && t_[p_] == '.') ++p_, digits(), is_float = true;
        if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
            ++p_;
            if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
            digits();
            is_float = true;
        }
        const std::string tok = t_.substr(start, p_ - start);
        if (!is_float) {
            if (tok[0] == '-') {
                long long v = 0;
                if (std::from_chars(tok.data(), tok.data() + tok.size(), v).ec == std::errc()) return Value(v);
            } else {
                unsigned long long v = 0;
                if (std::from_chars(tok.data(), tok.data() + tok.size(), v).ec == std::errc()) return Value(v);
            }
        }
        double d = 0.0;
        const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), d);
        if (r.ec != std::errc()) fail("number out of range");
        return Value(d);
    }

    const std::string& t_;
    size_t p_ = 0;
};

inline Value Value::parse(const std::string& text) { return Parser(text).document(); }

}  // namespace json
}  // namespace sfcb200
